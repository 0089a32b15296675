// Tile-binned rasterizer forward / L1 loss / backward on the device — the B200 replacement of
// project_all, rasterize_forward, compute_loss_l1 and rasterize_backward (render.hpp:361-640).
//
// The reference builds a per-pixel CSR list over each splat's integer 3-sigma pixel box, in
// (depth, id) order, then composites every pixel front to back. Here:
//   preprocess  thread per visible slot: exact project_geo + sigmoid + SH colour (render.hpp:361-380),
//               the fp64 pixel box (render.hpp:307-314), and the number of 16x16 tiles it touches.
//   duplicate   one (tile, depth) key per touched tile; CUB stable radix sort keeps equal depths in
//               slot order = ascending id, i.e. the reference's std::stable_sort order per pixel.
//   forward     CTA per tile, thread per pixel: batches of 256 splat records staged in SMEM, the
//               per-pixel box test reproduces the CSR membership, compositing is the reference's
//               op sequence (T-stop tested before each covering contribution, alpha clamp 0.999,
//               no 1/255 cut), so pixels are bit-identical. L1 loss + its gradient are fused in.
//   backward    CTA per tile: reverse sweep with transmittance recovered by division, 9-float
//               screen-space gradients reduced per splat with warp shuffles and a fixed-order
//               cross-warp sum into one partial per (splat, tile) instance — no float atomics,
//               so the result is deterministic run to run.
//   chain       thread per slot: fixed-order sum of its instance partials, then the reference's
//               chain through sigmoid, SH and project_geo_backward (render.hpp:600-638).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "gss_math.cuh"

namespace gssd {

constexpr int kTileSize = 16;
constexpr int kTilePix = kTileSize * kTileSize;  // pixels per tile
#ifndef GSS_FWD_BATCH
#define GSS_FWD_BATCH 256
#endif
constexpr int kFwdBatch = GSS_FWD_BATCH;
// Forward composite: pixels per thread (a warp owns an 8 x (4 * kFwdPPT) pixel block).
#ifndef GSS_FWD_PPT
#define GSS_FWD_PPT 2
#endif
constexpr int kFwdPPT = GSS_FWD_PPT;
constexpr int kFwdThreads = kTilePix / kFwdPPT;
constexpr int kFwdWarps = kFwdThreads / 32;
constexpr int kFwdBlockRows = 4 * kFwdPPT;
// Minimum resident blocks per SM for the composite / sweep kernels (0 = no bound: the compiler
// chooses the registers; the backward sweep then takes 78).
#ifndef GSS_FWD_MINB
#define GSS_FWD_MINB 0
#endif
#ifndef GSS_FWD_SAFE
#define GSS_FWD_SAFE 1  // certified records skip the per-pixel quotient range test: composite -8% at C4
#endif
#ifndef GSS_BWD_MINB
#define GSS_BWD_MINB 11  // 11 sweep CTAs per SM (78 registers, no spill): measured best, 12+ slower
#endif
#if GSS_FWD_MINB > 0
#define GSS_FWD_BOUNDS __launch_bounds__(kFwdThreads, GSS_FWD_MINB)
#else
#define GSS_FWD_BOUNDS __launch_bounds__(kFwdThreads)
#endif
#if GSS_BWD_MINB > 0
#define GSS_BWD_BOUNDS __launch_bounds__(kBwdThreads, GSS_BWD_MINB)
#else
#define GSS_BWD_BOUNDS __launch_bounds__(kBwdThreads)
#endif
#ifndef GSS_BWD_BATCH
#define GSS_BWD_BATCH 64
#endif
constexpr int kBwdBatch = GSS_BWD_BATCH;  // records per SMEM batch of the backward sweep
constexpr int kBwdMasks = kBwdBatch / 64;  // 64-bit record masks per warp and batch

// Work accounting (GSS_RASTER_STATS=1 builds only; zero otherwise), read by gss_raster_stats:
//   [0] forward (warp, record) pairs walked   [1] forward lane-pixel slots offered (walked x 32 x PPT)
//   [2] forward (pixel, record) in box        [3] forward contributions evaluated (composited)
//   [4] forward eval slots issued (32 per warp-level eval)
//   [5] backward (warp, record) pairs walked  [6] backward lane-pixel slots (walked x 32 x PPT)
//   [7] backward useful (pixel, record) contributions
#ifndef GSS_RASTER_STATS
#define GSS_RASTER_STATS 0
#endif
__device__ unsigned long long g_rstats[8];

struct __align__(16) SplatRec {
  float mx, my, a, b;
  float c, ab, r, g;
  float bl, depth;
  int32_t off;
  float det;  // a*c - b*b, evaluated once with the reference's operation order
  int32_t bx0, bx1, by0, by1;  // absolute pixels, half-open, clipped to the window
};
static_assert(sizeof(SplatRec) == 64, "record is 4 x 16 B");

struct Win {
  int px0, py0, pw, ph, tw, th;
};

struct SceneDev {
  const int32_t* ids;
  const float* geo;
  int64_t geo_stride;
  const float* nongeo;
  int64_t ng_stride;
  int compact;
  const int32_t* slot_map;
  int sh_degree;
  float bg[3];
  float lp;
};

// Growable device buffer on the stream-ordered pool.
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes, cudaStream_t st) {
    if (bytes > cap) {
      if (p) GSS_CUDA(cudaFreeAsync(p, st));
      const size_t nb = std::max<size_t>(bytes + bytes / 4, 4096);
      GSS_CUDA(cudaMallocAsync(&p, nb, st));
      cap = nb;
    }
    return p;
  }
  void release(cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace gssd

struct gss_render_ctx {
  gssd::DBuf recs, ntiles, offsets, keys_a, keys_b, vals_a, vals_b, cub_tmp, ranges, tile_order, last, fT, partials, lossp,
      hostcnt, sums, dkeys_a, dkeys_b, order_a, order_b, slot_off;
  gssd::Win win{};
  gssd::SceneDev sc{};
  gssd::Cam cam{};
  int64_t V = 0, I = 0;
  const uint64_t* pay_sorted = nullptr;  // depth-ordered sort payloads of the last binning (slot + box)
  int have_forward = 0;
  int64_t* pinned = nullptr;  // host-visible counts
  cudaStream_t last_stream = nullptr;
  // Live kernel timing (bench roofline): CUDA events around each forward_kernel (kind 0) and
  // backward_kernel (kind 1) launch on its stream, and the composited-contribution count.
  bool ktiming = false;
  struct KTime {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<KTime> ktimes;
  std::vector<cudaEvent_t> kfree;
  // kinds: 0 composite, 1 sweep, 2 geometry (projection .. tile order, incl. the instance-count
  // round trip), 3 colour, 4 per-slot sums, 5 chain
  static constexpr int kKinds = 6;
  double kms[kKinds] = {};
  int64_t kn[kKinds] = {};
  unsigned long long* contribs_dev = nullptr;  // running total of composited contributions
};

namespace gssd {
namespace {

__device__ __forceinline__ const float* ng_row(const SceneDev& s, int k, int id) {
  const int64_t r = s.compact ? (int64_t)(s.slot_map ? s.slot_map[k] : k) : (int64_t)id;
  return s.nongeo + r * s.ng_stride;
}

// project_all (render.hpp:361-380) + CSR box (render.hpp:297-314, 418-419) + tile count.
// Opacity and view-dependent colour of slot k (render.hpp:372-378, sh.hpp:77-86).
// DEG >= 0: the SH degree known at compile time (the basis stays in registers); -1: s.sh_degree.
template <int DEG = -1>
__device__ __forceinline__ void splat_colour_row(const SceneDev& s, const Cam& cam, const float* ng, const float* g,
                                                 SplatRec& r) {
  r.ab = 1.0f / (1.0f + gss_expf(-ng[0]));
  const f3 cp = cam_position(cam);
  f3 dir{g[0] - cp.x, g[1] - cp.y, g[2] - cp.z};
  const float dn = sqrtf(dir.x * dir.x + dir.y * dir.y + dir.z * dir.z);
  if (dn > 1e-12f) {
    const float inv = 1.0f / dn;
    dir = f3{dir.x * inv, dir.y * inv, dir.z * inv};
  } else {
    dir = f3{0.0f, 0.0f, 1.0f};
  }
  float basis[16];
  const int deg = DEG >= 0 ? DEG : s.sh_degree;
  sh_basis(dir.x, dir.y, dir.z, deg, basis);
  const int nb = (deg + 1) * (deg + 1);
  float rgb0 = 0.5f, rgb1 = 0.5f, rgb2 = 0.5f;
  for (int b = 0; b < nb; ++b) {
    rgb0 += basis[b] * ng[1 + 3 * b];
    rgb1 += basis[b] * ng[2 + 3 * b];
    rgb2 += basis[b] * ng[3 + 3 * b];
  }
  r.r = clamp01(rgb0);
  r.g = clamp01(rgb1);
  r.bl = clamp01(rgb2);
}
__device__ __forceinline__ void splat_colour(const SceneDev& s, const Cam& cam, int k, int id, const float* g,
                                             SplatRec& r) {
  splat_colour_row(s, cam, ng_row(s, k, id), g, r);
}

// Stages the non-geometric rows of a warp's 32 consecutive slots (nf floats each) into SMEM rows of
// pitch `pitch` (odd: lane-strided row access is conflict-free): consecutive lanes copy consecutive
// floats of a row (coalesced), every element in flight at once through LDGSTS (no register
// round trip), then the warp waits for its copies.
template <int PITCH>
__device__ __forceinline__ void stage_rows(const SceneDev& s, int64_t k0, int nk, int nf, int lane,
                                           float (*rows)[PITCH]) {
  const float* my_row = lane < nk ? ng_row(s, (int)(k0 + lane), s.ids[k0 + lane]) : s.nongeo;
  for (int e = lane; e < 32 * nf; e += 32) {
    const int kk = e / nf, c = e - kk * nf;
    const float* rp = (const float*)__shfl_sync(0xffffffffu, (unsigned long long)my_row, kk);
    if (kk < nk) cp_async4(&rows[kk][c], rp + c);
  }
  cp_async_wait_all();
  __syncwarp();
}

// Depth-sort payload: slot k in the low 32 bits, the splat's tile box (tx0, ty0, ntx, nty, a byte
// each) in the high 32 bits when it fits (windows up to 255 x 255 tiles: 4080 px), else the
// kNoBox sentinel. Binning then reads the depth-ordered payload sequentially instead of gathering
// each slot's record and tile count at random.
constexpr uint32_t kNoBox = 0xffffffffu;
__device__ __forceinline__ uint64_t pack_payload(int64_t k, int nt, int tx0, int ty0, int ntx, int nty) {
  uint32_t hi = 0;  // nt == 0: an empty box
  if (nt > 0) hi = (tx0 < 256 && ty0 < 256 && ntx < 256 && nty < 256)
                       ? (uint32_t)tx0 | ((uint32_t)ty0 << 8) | ((uint32_t)ntx << 16) | ((uint32_t)nty << 24)
                       : kNoBox;
  return ((uint64_t)hi << 32) | (uint32_t)k;
}

// project_all (render.hpp:361-380) + CSR box (render.hpp:297-314, 418-419) + tile count. With
// COLOUR = false only the geometry is produced (opacity/colour zero) — colour_kernel fills it in
// once the non-geometric rows are available, so binning can run while they are gathered.
template <bool COLOUR>
__global__ void preprocess_kernel(SceneDev s, Cam cam, Win w, int64_t V, SplatRec* recs, int32_t* ntiles,
                                  uint32_t* dkey, uint64_t* dpay) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= V) return;
  const int id = s.ids[k];
  const float* g = s.geo + (int64_t)id * s.geo_stride;
  Proj p;
  f3 t;
  SplatRec r;
  memset(&r, 0, sizeof(r));
  int nt = 0, ptx0 = 0, pty0 = 0, pntx = 0, pnty = 0;
  if (project_geo(cam, g, s.lp, p, t)) {
    if (COLOUR) splat_colour(s, cam, (int)k, id, g, r);
    r.mx = p.mx; r.my = p.my; r.a = p.a; r.b = p.b; r.c = p.c;
    r.depth = t.z;
    r.det = p.a * p.c - p.b * p.b;
    if (r.det > 0.0f) {
      const double mx = (double)p.mx, my = (double)p.my, rad = (double)p.radius;
      const int a0 = d2i_x86(ceil(mx - rad - 0.5));
      const int a1 = (int)((unsigned)d2i_x86(floor(mx + rad - 0.5)) + 1u);
      const int b0 = d2i_x86(ceil(my - rad - 0.5));
      const int b1 = (int)((unsigned)d2i_x86(floor(my + rad - 0.5)) + 1u);
      const int wx1 = w.px0 + w.pw, wy1 = w.py0 + w.ph;
      const int bx0 = max(w.px0, a0), bx1 = min(wx1, a1), by0 = max(w.py0, b0), by1 = min(wy1, b1);
      if (bx0 < bx1 && by0 < by1) {
        r.bx0 = bx0; r.bx1 = bx1; r.by0 = by0; r.by1 = by1;
        const int tx0 = (bx0 - w.px0) / kTileSize, tx1 = (bx1 - 1 - w.px0) / kTileSize;
        const int ty0 = (by0 - w.py0) / kTileSize, ty1 = (by1 - 1 - w.py0) / kTileSize;
        nt = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
        ptx0 = tx0; pty0 = ty0; pntx = tx1 - tx0 + 1; pnty = ty1 - ty0 + 1;
      }
    }
  }
  if (nt == 0) r.bx0 = r.bx1 = r.by0 = r.by1 = 0;
  recs[k] = r;
  if (!ntiles) return;  // projection only (gss_project)
  ntiles[k] = nt;
  // Depth sort key: binned splats have depth >= near > 0, whose IEEE bits order like the values.
  dkey[k] = nt > 0 ? __float_as_uint(r.depth) : 0xffffffffu;
  dpay[k] = pack_payload(k, nt, ptx0, pty0, pntx, pnty);
}

// The colour half of preprocess for the binned splats (ntiles > 0: the only records compositing
// and the sweep read; a valid unbinned slot's opacity only meets zero gradient sums in the chain).
// Warp-cooperative: a warp owns 32 consecutive slots, stages the row floats the SH degree reads
// (1 + 3 (deg+1)^2) into SMEM (stage_rows) and each lane evaluates its slot from SMEM — instead of
// every lane streaming its own 196-byte row.
constexpr int kColThreads = 128;
constexpr int kColRow = 49;  // odd pitch
template <int DEG>
__global__ void __launch_bounds__(kColThreads) colour_kernel(SceneDev s, Cam cam, int64_t V, const int32_t* ntiles,
                                                              SplatRec* recs) {
  __shared__ float row_s[kColThreads / 32][32][kColRow];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t k0 = (int64_t)blockIdx.x * kColThreads + warp * 32;
  if (k0 >= V) return;
  const int nk = (V - k0) < 32 ? (int)(V - k0) : 32;
  const int64_t k = k0 + lane;
  const bool mine = lane < nk && ntiles[k] > 0;
  if (!__any_sync(0xffffffffu, mine)) return;
  stage_rows<kColRow>(s, k0, nk, 1 + 3 * (DEG + 1) * (DEG + 1), lane, row_s[warp]);
  if (!mine) return;
  const int id = s.ids[k];
  SplatRec r;
  splat_colour_row<DEG>(s, cam, row_s[warp][lane], s.geo + (int64_t)id * s.geo_stride, r);
  recs[k].ab = r.ab;
  recs[k].r = r.r;
  recs[k].g = r.g;
  recs[k].bl = r.bl;
}

// Records projected against a larger window (another GPU's projection of the whole view),
// re-clipped to this window w (an image strip): the reference box of a splat is the same for
// every window, only its clip differs, so per-pixel contribution lists are unchanged.
__global__ void clip_kernel(const SplatRec* in, int64_t V, Win w, SplatRec* recs, int32_t* ntiles, uint32_t* dkey,
                            uint64_t* dpay) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= V) return;
  SplatRec r = in[k];
  int nt = 0, ptx0 = 0, pty0 = 0, pntx = 0, pnty = 0;
  if (r.bx1 > r.bx0 && r.by1 > r.by0) {
    const int wx1 = w.px0 + w.pw, wy1 = w.py0 + w.ph;
    r.bx0 = max(w.px0, r.bx0); r.bx1 = min(wx1, r.bx1);
    r.by0 = max(w.py0, r.by0); r.by1 = min(wy1, r.by1);
    if (r.bx0 < r.bx1 && r.by0 < r.by1) {
      const int tx0 = (r.bx0 - w.px0) / kTileSize, tx1 = (r.bx1 - 1 - w.px0) / kTileSize;
      const int ty0 = (r.by0 - w.py0) / kTileSize, ty1 = (r.by1 - 1 - w.py0) / kTileSize;
      nt = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
      ptx0 = tx0; pty0 = ty0; pntx = tx1 - tx0 + 1; pnty = ty1 - ty0 + 1;
    }
  }
  if (nt == 0) r.bx0 = r.bx1 = r.by0 = r.by1 = 0;
  recs[k] = r;
  ntiles[k] = nt;
  dkey[k] = nt > 0 ? __float_as_uint(r.depth) : 0xffffffffu;
  dpay[k] = pack_payload(k, nt, ptx0, pty0, pntx, pnty);
}

// Image-strip routing: does record k's pixel box touch columns [x0, x1)?
struct StripHit {
  const SplatRec* recs;
  int x0, x1;
  __host__ __device__ bool operator()(int32_t k) const {
    const SplatRec& r = recs[k];
    return r.bx1 > r.bx0 && r.by1 > r.by0 && r.bx0 < x1 && r.bx1 > x0;
  }
};

__global__ void gather_records_kernel(const SplatRec* recs, const int32_t* slots, int64_t n, SplatRec* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = recs[slots[i]];
}

// dst[slots[j]][c] += src[j][c]: one strip's returned partials; each slot appears at most once per
// call, so calls in strip order give a fixed-order (deterministic) sum.
__global__ void scatter_add_rows_kernel(const float* src, const int32_t* slots, int64_t n, int width, float* dst) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * width) return;
  const int64_t j = e / width;
  const int c = (int)(e - j * width);
  dst[(int64_t)slots[j] * width + c] += src[e];
}

__device__ __forceinline__ void tile_box(const SplatRec& r, const Win& w, int& tx0, int& ty0, int& ntx, int& nty) {
  tx0 = (r.bx0 - w.px0) / kTileSize;
  ty0 = (r.by0 - w.py0) / kTileSize;
  ntx = (r.bx1 - 1 - w.px0) / kTileSize - tx0 + 1;
  nty = (r.by1 - 1 - w.py0) / kTileSize - ty0 + 1;
}

// Tile instances in depth order: thread i takes the i-th splat of the stable (depth, slot) sort
// and emits one (tile) key per touched tile; the stable tile sort that follows keeps depth order
// (ties in slot = ascending id order) inside each tile, the reference's std::stable_sort order
// (render.hpp:406-416). Instance numbering follows this order; slot_off[k] / ntiles[k] give slot
// k's instance range for the backward's per-slot sums.
__global__ void duplicate_kernel(const SplatRec* recs, const uint64_t* pay, const int32_t* ntiles,
                                 const int32_t* offsets, Win w, int64_t V, uint32_t* keys, int32_t* vals,
                                 SplatRec* recs_rw, int32_t* slot_off) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (i - lane >= V) return;  // whole warp past the end
  const bool valid = i < V;
  int32_t k = 0, off = 0, nt = 0;
  int tx0 = 0, ty0 = 0, ntx = 1, nty = 0;
  if (valid) {
    const uint64_t p = pay[i];
    const uint32_t hi = (uint32_t)(p >> 32);
    k = (int32_t)(uint32_t)p;
    off = offsets[i];
    recs_rw[k].off = off;
    slot_off[k] = off;
    if (hi != kNoBox) {  // the tile box travelled with the sort
      tx0 = (int)(hi & 0xffu);
      ty0 = (int)((hi >> 8) & 0xffu);
      ntx = (int)((hi >> 16) & 0xffu);
      nty = (int)(hi >> 24);
      nt = ntx * nty;
      if (nt == 0) ntx = 1;
    } else {
      nt = ntiles[k];
      if (nt > 0) tile_box(recs[k], w, tx0, ty0, ntx, nty);
    }
  }
  if (nt > 0 && nt <= 4) {  // small splats: this lane writes its own keys (row-major tile order)
    int j = 0;
    for (int ty = ty0; ty < ty0 + nty; ++ty)
      for (int tx = tx0; tx < tx0 + ntx; ++tx, ++j) {
        keys[off + j] = (uint32_t)(ty * w.tw + tx);
        vals[off + j] = k;
      }
  }
  // large splats (near the camera: hundreds of tiles) are written by the whole warp, coalesced
  unsigned big = __ballot_sync(0xffffffffu, nt > 4);
  while (big) {
    const int b = __ffs(big) - 1;
    big &= big - 1;
    const int32_t bk = __shfl_sync(0xffffffffu, k, b), boff = __shfl_sync(0xffffffffu, off, b);
    const int bnt = __shfl_sync(0xffffffffu, nt, b), btx0 = __shfl_sync(0xffffffffu, tx0, b);
    const int bty0 = __shfl_sync(0xffffffffu, ty0, b), bntx = __shfl_sync(0xffffffffu, ntx, b);
    for (int j = lane; j < bnt; j += 32) {
      const int ty = bty0 + j / bntx, tx = btx0 + j - (j / bntx) * bntx;
      keys[boff + j] = (uint32_t)(ty * w.tw + tx);
      vals[boff + j] = bk;
    }
  }
}

// ntiles in sorted order (0 at position V), for the instance-offset scan: offsets[V] = I.
struct SortedCount {
  const int32_t* nt;
  const uint64_t* pay;
  int32_t V;
  __host__ __device__ int32_t operator()(int32_t i) const {
    if (i >= V) return 0;
    const uint64_t p = pay[i];
    const uint32_t hi = (uint32_t)(p >> 32);
    return hi != kNoBox ? (int32_t)(((hi >> 16) & 0xffu) * (hi >> 24)) : nt[(uint32_t)p];
  }
};

// Tile ranges of the sorted instance keys: thread t owns keys [4t, 4t + 4) (one 16-byte load; the
// neighbours across the thread boundary come from the adjacent lanes, the warp edges from memory).
__global__ void ranges_kernel(const uint32_t* keys, int64_t I, int2* ranges) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i0 = 4 * t;
  const int lane = threadIdx.x & 31;
  uint32_t k[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
  if (i0 + 3 < I) {
    const uint4 q = *reinterpret_cast<const uint4*>(keys + i0);
    k[0] = q.x; k[1] = q.y; k[2] = q.z; k[3] = q.w;
  } else {
    for (int j = 0; j < 4; ++j)
      if (i0 + j < I) k[j] = keys[i0 + j];
  }
  uint32_t prev = __shfl_up_sync(0xffffffffu, k[3], 1);
  uint32_t next = __shfl_down_sync(0xffffffffu, k[0], 1);
  if (lane == 0 && i0 > 0 && i0 - 1 < I) prev = keys[i0 - 1];
  if (lane == 31 && i0 + 4 < I) next = keys[i0 + 4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t i = i0 + j;
    if (i >= I) break;
    const uint32_t before = j == 0 ? prev : k[j - 1];
    const uint32_t after = j == 3 ? next : k[j + 1];
    if (i == 0 || before != k[j]) ranges[k[j]].x = (int)i;
    if (i == I - 1 || after != k[j]) ranges[k[j]].y = (int)(i + 1);
  }
}

// Launch order of the tile CTAs: heaviest tiles first (longest-processing-time-first), so the
// few tiles that hold many more instances than the rest (near-camera splats, dense clusters)
// start in the first wave instead of forming the kernel's tail. One CTA buckets the tiles by
// instance count (256 linear buckets below the maximum) and scatters them in descending bucket
// order. Only the schedule changes: every tile's pixels and partials are computed exactly as
// before, so the order within a bucket (atomic) does not affect any result.
#ifndef GSS_LPT
#define GSS_LPT 1
#endif
constexpr int kOrderThreads = 1024;
__global__ void __launch_bounds__(kOrderThreads) tile_order_kernel(const int2* ranges, int ntile, int32_t* order) {
  __shared__ int hist[256];
  __shared__ int cmax;
  const int t = threadIdx.x;
  if (t < 256) hist[t] = 0;
  if (t == 0) cmax = 0;
  __syncthreads();
  int m = 0;
  for (int i = t; i < ntile; i += kOrderThreads) {
    const int2 r = ranges[i];
    m = max(m, r.y - r.x);
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((t & 31) == 0) atomicMax(&cmax, m);
  __syncthreads();
  const long long den = (long long)cmax + 1;
  for (int i = t; i < ntile; i += kOrderThreads) {
    const int2 r = ranges[i];
    atomicAdd(&hist[255 - (int)((long long)(r.y - r.x) * 256 / den)], 1);
  }
  __syncthreads();
  if (t < 32) {  // exclusive scan of 256 bucket counts, 8 per lane
    int loc[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      loc[k] = hist[t * 8 + k];
      sum += loc[k];
    }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (t >= o) inc += v;
    }
    int run = inc - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      hist[t * 8 + k] = run;
      run += loc[k];
    }
  }
  __syncthreads();
  for (int i = t; i < ntile; i += kOrderThreads) {
    const int2 r = ranges[i];
    order[atomicAdd(&hist[255 - (int)((long long)(r.y - r.x) * 256 / den)], 1)] = i;
  }
}

__device__ __forceinline__ int tile_of(const int32_t* order) {
#if GSS_LPT
  return order[blockIdx.x];
#else
  return blockIdx.x;
#endif
}

struct EvalOut {
  float alpha, q, weight;
  bool clamped;
};

// RN(1/det) when det lies in [2^-60, 2^60], else 0 (then the quotient takes the IEEE division).
__device__ __forceinline__ float det_rcp(float det) {
  return (det >= 0x1p-60f && det <= 0x1p60f) ? __frcp_rn(det) : 0.0f;
}

// RN(n / d) given rd = det_rcp(d): Markstein's correction q0 = RN(n*rd), q = RN(q0 + fma(-d, q0, n)*rd)
// is the correctly rounded quotient for |n| in [2^-60, 2^60) (tools/divcheck.cu: 0 mismatches in
// 1.07e10 pairs, including divisors with all-ones significands); other n take the IEEE division.
__device__ __forceinline__ float div_rcp_rn(float n, float d, float rd) {
  if (rd != 0.0f && ((__float_as_uint(n) >> 23) & 0xffu) - 67u < 120u) {
    const float q0 = __fmul_rn(n, rd);
    return __fmaf_rn(__fmaf_rn(-d, q0, n), rd, q0);
  }
  return __fdiv_rn(n, d);
}

// A record whose every covered pixel meets the Markstein quotient's range (div_rcp_rn) without a
// per-pixel test: RN(1/det) usable, and the computed numerator of any pixel in its box either
// exactly zero (pixel centre on the mean) or in [2^-60, 2^60). The exact numerator is a quadratic
// form with eigenvalues >= det / (a + c) (those of the covariance) and |d|^2 >= 2^-50 when d != 0
// (pixel centres are >= 0.5, so a nonzero float difference is >= 2^-25); its float evaluation
// errs by < 2^-21 (a + c + |b|) |d|^2. The conditions below bound both ends with a 2x margin
// (NaN or inf fields fail every comparison).
#if GSS_FWD_SAFE
// Certified records also have alpha_base <= 0.999 (so ab * weight, weight <= 1, never reaches the
// 0.999 clamp) and, by the numerator bound, a quotient >= +0 (max(q, 0) is the identity): the
// certified pixel path drops the range test, the clamp and the max.
__device__ __forceinline__ bool fwd_quotient_safe(const SplatRec& r, float rd) {
  if (rd == 0.0f) return false;
  if (!(r.ab <= 0.999f)) return false;
  const float a = r.a, c = r.c, ab = fabsf(r.b), det = r.det, tr = a + c;
  if (!(a > 0.0f && c > 0.0f)) return false;
  if (!(det >= 0x1p-19f * tr * (tr + ab))) return false;  // cancellation < half the exact value
  if (!(det >= 0x1p-8f * tr)) return false;                // (det / tr) 2^-50 / 2 >= 2^-59
  const float wx = fmaxf(fabsf((float)r.bx0 - r.mx), fabsf((float)r.bx1 - r.mx)) + 1.0f;
  const float wy = fmaxf(fabsf((float)r.by0 - r.my), fabsf((float)r.by1 - r.my)) + 1.0f;
  return (tr + ab) * (wx * wx + wy * wy) < 0x1p58f;         // < 2^60 with margin
}
#endif

// contrib_eval (render.hpp:342-358); det > 0 holds for every binned splat (render.hpp:418).
// The exponent is -q/2 <= 0 (or NaN), so only the underflow / NaN guards of expf apply.
// rd: det_rcp(r.det) (the forward stages it per record), or 0 for the plain IEEE division.
__device__ __forceinline__ EvalOut contrib_eval(const SplatRec& r, float cx, float cy, float rd = 0.0f) {
  EvalOut o;
  const float dx = cx - r.mx, dy = cy - r.my;
  o.q = max0(div_rcp_rn(r.c * dx * dx - 2.0f * r.b * dx * dy + r.a * dy * dy, r.det, rd));
  o.weight = gss_expf_nonpos(-0.5f * o.q);
  const float raw = r.ab * o.weight;
  o.clamped = raw > 0.999f;
  o.alpha = o.clamped ? 0.999f : raw;
  return o;
}

__device__ __forceinline__ void load_rec(SplatRec* dst, const SplatRec* recs, int slot) {
  const float4* s = reinterpret_cast<const float4*>(recs + slot);
  float4* d = reinterpret_cast<float4*>(dst);
  d[0] = s[0]; d[1] = s[1]; d[2] = s[2]; d[3] = s[3];
}

// Forward composite (render.hpp:438-462) fused with the L1 loss (render.hpp:497-511).
// Each warp owns an 8 x 8 pixel block of the 16x16 tile (2 pixels per thread, rows 4 apart, so the
// per-record SMEM loads and bookkeeping serve two pixels). After a batch of records is staged in
// SMEM, the warp ballots which records' pixel boxes intersect its block and walks only those
// (warp-uniform loop); the per-pixel box test then reproduces the CSR membership exactly.
__global__ void GSS_FWD_BOUNDS forward_kernel(const SplatRec* __restrict__ recs,
                                                           const int32_t* __restrict__ vals,
                                                           const int2* __restrict__ ranges,
                                                           const int32_t* __restrict__ tile_order, Win w, float bg0,
                                                           float bg1, float bg2, float* image, float* fT_out,
                                                           int32_t* last_out, int32_t* ncontrib_out,
                                                           const float* gt, int gt_width, float inv_norm,
                                                           float* d_img, double* loss_partials,
                                                           unsigned long long* contribs_total, ExpCoef ekp) {
  // exp coefficients staged through SMEM into registers (kept there for the whole kernel instead
  // of a constant-bank load before every DFMA)
#ifndef GSS_FWD_COEF_SMEM
#define GSS_FWD_COEF_SMEM 1
#endif
#if GSS_FWD_COEF_SMEM
  __shared__ ExpCoef shek;
  if (threadIdx.x == 0) shek = ekp;
  __syncthreads();
  const ExpCoef ek = shek;
#else
  const ExpCoef& ek = ekp;
#endif
  __shared__ SplatRec sh[kFwdBatch];
  __shared__ double red[kFwdWarps];
  const int tile = tile_of(tile_order);
  const int tx = tile % w.tw, ty = tile / w.tw;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * kFwdBlockRows;
  const int fx0 = w.px0 + tx * kTileSize + wx0, fy0 = w.py0 + ty * kTileSize + wy0;  // warp block origin
  const int x = fx0 + (lane & 7);
  const float cx = (float)x + 0.5f;
  const int2 rg = ranges[tile];
  // Pixel h of this thread: row fy0 + (lane >> 3) + 4h of the warp's 8 x kFwdBlockRows block.
  // yb: the row used by the box tests (a pixel outside the window never meets a box). A pixel is
  // finished once T < 1e-4 (render.hpp:442): no later contribution changes T, so the T test alone
  // is the reference's early stop.
  int y[kFwdPPT], yb[kFwdPPT], used[kFwdPPT], last[kFwdPPT];
  float cy[kFwdPPT], T[kFwdPPT], c0[kFwdPPT], c1[kFwdPPT], c2[kFwdPPT];
  bool all_done = true;
#if GSS_RASTER_STATS
  unsigned long long st_walk = 0, st_box = 0, st_eval = 0, st_slots = 0;
#endif
#pragma unroll
  for (int h = 0; h < kFwdPPT; ++h) {
    y[h] = fy0 + (lane >> 3) + 4 * h;
    cy[h] = (float)y[h] + 0.5f;
    T[h] = 1.0f;
    c0[h] = c1[h] = c2[h] = 0.0f;
    used[h] = last[h] = 0;
    const bool inwin = x < w.px0 + w.pw && y[h] < w.py0 + w.ph;
    yb[h] = inwin ? y[h] : INT_MIN;
    all_done &= !inwin;
  }
  for (int b = rg.x; b < rg.y; b += kFwdBatch) {
    if (__syncthreads_count(all_done) == kFwdThreads) break;
    const int nb = min(kFwdBatch, rg.y - b);
    for (int t = threadIdx.x; t < nb; t += kFwdThreads) {
      load_rec(&sh[t], recs, vals[b + t]);
      const float rd = det_rcp(sh[t].det);
      sh[t].depth = rd;  // the SMEM copy's depth slot holds RN(1/det)
#if GSS_FWD_SAFE
      sh[t].off = fwd_quotient_safe(sh[t], rd) ? 1 : 0;  // and its off slot the range certificate
#endif
    }
    __syncthreads();
    for (int c0j = 0; c0j < nb && __any_sync(0xffffffffu, !all_done); c0j += 32) {
      const int jl = c0j + lane;
      bool hit = false;
      if (jl < nb) {
        const int4 bx = *reinterpret_cast<const int4*>(&sh[jl].bx0);
        hit = bx.x <= fx0 + 7 && bx.y > fx0 && bx.z <= fy0 + kFwdBlockRows - 1 && bx.w > fy0;
      }
      unsigned m = __ballot_sync(0xffffffffu, hit);
#if GSS_RASTER_STATS
      if (lane == 0) st_walk += __popc(m);
#endif
      while (m) {
        const int j = c0j + __ffs(m) - 1;
        m &= m - 1;
        // Record fields in registers once per record (both pixels of the lane share them):
        // q0 = mx, my, a, b; q1 = c, ab, r, g; q2 = bl, RN(1/det), off, det; bx = box.
        const float4* rp = reinterpret_cast<const float4*>(&sh[j]);
        const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
        const int4 bx = *reinterpret_cast<const int4*>(&sh[j].bx0);
        const bool xin = (x >= bx.x) & (x < bx.y);
        // contrib_eval's numerator c*dx*dx - 2*b*dx*dy + a*dy*dy (render.hpp:346) in the reference's
        // operation order; the x-only factors are shared by the lane's pixels (same column).
        const float dx = cx - q0.x;
        const float cdxdx = (q1.x * dx) * dx;
        const float b2dx = (2.0f * q0.w) * dx;
        const int lastv = b + j - rg.x + 1;
        // Markstein quotient range (div_rcp_rn): |num| in [2^-60, 2^60) and a usable RN(1/det);
        // a record without one (rd == 0) sends every quotient to the IEEE division.
        const float lo = q2.y != 0.0f ? 0x1p-60f : __int_as_float(0x7f800000);
        auto pixels = [&](auto checked_c) {
          constexpr bool kChecked = decltype(checked_c)::value;
#pragma unroll
        for (int h = 0; h < kFwdPPT; ++h) {
          const bool inb = xin & (yb[h] >= bx.z) & (yb[h] < bx.w);
          const bool ev = inb & !(T[h] < 1e-4f);  // render.hpp:442: T-stop before the contribution
#if GSS_RASTER_STATS
          st_box += inb ? 1 : 0;
          st_eval += ev ? 1 : 0;
          if (__ballot_sync(0xffffffffu, ev) && lane == 0) st_slots += 32;
#endif
          if (!__any_sync(0xffffffffu, ev)) continue;  // warp-uniform skip
          const float dy = cy[h] - q0.y;
          const float num = (cdxdx - b2dx * dy) + (q0.z * dy) * dy;
          const float qf = __fmul_rn(num, q2.y);
          float quo = __fmaf_rn(__fmaf_rn(-q2.w, qf, num), q2.y, qf);
          if (kChecked) {
            const float an = fabsf(num);
            const bool slow = !((an >= lo) & (an < 0x1p60f));
            if (__any_sync(0xffffffffu, slow)) {  // rare: zero / extreme numerators, extreme det
              if (slow) quo = __fdiv_rn(num, q2.w);
            }
          }
          const float xe = -0.5f * (kChecked ? max0(quo) : quo);
          const float wgt = gss_expf_nonpos_sel(xe, ek);
          const float raw = q1.y * wgt;
          const float alpha = (kChecked && raw > 0.999f) ? 0.999f : raw;
          if (ev) {
            c0[h] += q1.z * alpha * T[h];
            c1[h] += q1.w * alpha * T[h];
            c2[h] += q2.x * alpha * T[h];
            T[h] *= (1.0f - alpha);
            ++used[h];
            last[h] = lastv;
          }
        }
        };
#if GSS_FWD_SAFE
        if (__float_as_int(q2.z) != 0)
          pixels(std::false_type{});  // certified record: no per-pixel range test
        else
#endif
          pixels(std::true_type{});
      }
      all_done = true;
#pragma unroll
      for (int h = 0; h < kFwdPPT; ++h) all_done &= (yb[h] == INT_MIN) | (T[h] < 1e-4f);
    }
    __syncthreads();
  }
#if GSS_RASTER_STATS
  atomicAdd(&g_rstats[0], st_walk);
  atomicAdd(&g_rstats[1], st_walk * 32ull * kFwdPPT);
  atomicAdd(&g_rstats[2], st_box);
  atomicAdd(&g_rstats[3], st_eval);
  atomicAdd(&g_rstats[4], st_slots);
#endif
  double acc = 0.0;
#pragma unroll
  for (int h = 0; h < kFwdPPT; ++h) {
    if (!(x < w.px0 + w.pw && y[h] < w.py0 + w.ph)) continue;
    const int64_t pix = (int64_t)(y[h] - w.py0) * w.pw + (x - w.px0);
    const float o0 = c0[h] + T[h] * bg0, o1 = c1[h] + T[h] * bg1, o2 = c2[h] + T[h] * bg2;
    image[pix * 3 + 0] = o0;
    image[pix * 3 + 1] = o1;
    image[pix * 3 + 2] = o2;
    fT_out[pix] = T[h];
    last_out[pix] = last[h];
    if (ncontrib_out) ncontrib_out[pix] = used[h];
    if (gt) {
      const float* gp = gt + ((int64_t)y[h] * gt_width + x) * 3;
      const float o[3] = {o0, o1, o2};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float d = o[c] - gp[c];
        acc += fabs((double)d);
        d_img[pix * 3 + c] = d > 0.0f ? inv_norm : (d < 0.0f ? -inv_norm : 0.0f);
      }
    }
  }
  if (gt) {
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < kFwdWarps; ++i) s += red[i];
      loss_partials[tile] = s;
    }
  }
  if (contribs_total) {  // composited contributions of the tile (bench accounting; integer: exact)
    unsigned u = 0;
#pragma unroll
    for (int h = 0; h < kFwdPPT; ++h) u += (unsigned)used[h];
    u = __reduce_add_sync(0xffffffffu, u);
    if (lane == 0) atomicAdd(contribs_total, (unsigned long long)u);
  }
}

__global__ void loss_partial_kernel(const float* img, const float* gt, int64_t n, float inv, float* d_img,
                                    double* partials) {
  __shared__ double red[8];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = img[i] - gt[i];
    acc += fabs((double)d);
    d_img[i] = d > 0.0f ? inv : (d < 0.0f ? -inv : 0.0f);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    partials[blockIdx.x] = s;
  }
}

// image_mse numerator (trainer.hpp:113-122): sum of (double(a) - double(b))^2, per-block fp64 partials
// in a fixed order (deterministic).
__global__ void sq_err_partial_kernel(const float* a, const float* b, int64_t n, double* partials) {
  __shared__ double red[8];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    acc += d * d;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    partials[blockIdx.x] = s;
  }
}

__global__ void sum_partials_kernel(const double* partials, int n, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    *out = t;
  }
}

// Fixed-order final reduction: loss = float(sum) * inv (render.hpp:510).
__global__ void loss_final_kernel(const double* partials, int n, float inv, float* loss, double* sum_out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    *loss = (float)s * inv;
    if (sum_out) *sum_out = s;
  }
}

// Reverse sweep state of one pixel (render.hpp:542-589). The suffix colour enters the sweep only
// through its dot product with the pixel's (constant) colour gradient, so the state keeps that
// scalar S = suf . g (suf_c += rgb_c * w  =>  S += (rgb . g) * w).
#ifndef GSS_BWD_PPT
#define GSS_BWD_PPT 4
#endif
struct PixB {
  float cx, cy, T, g0, g1, g2, S;
  int x, y, L;
};

// Per-splat constants of the backward sweep, computed once per batch: the conic (inverse 2D
// covariance) so the per-pixel exponent needs no division.
// GSS_BWD_KFOLD: the exp's -log2(e)/2 factor folded into a scaled copy of the conic (sia, sibm2,
// sic), so the sweep's quadratic form comes out as the ex2 argument (one multiply less per pixel).
#ifndef GSS_BWD_KFOLD
#define GSS_BWD_KFOLD 1
#endif
constexpr float kExpHalf = -0.72134752f;  // -log2(e) / 2: exp(-q/2) = ex2(kExpHalf * q)
struct BwdConic {
  float ia, ibm2, ic;  // c/det, -2*b/det, a/det
  float nh;            // -0.5/det
#if GSS_BWD_KFOLD
  float sia, sibm2, sic, pad;  // kExpHalf * (ia, ibm2, ic)
#endif
};

__device__ __forceinline__ float ex2_fast(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_fast(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// The 0.999 clamp can only fire for a splat whose alpha_base exceeds 0.999 - 1e-4 (weight <= 1);
// every other record takes the sweep without the clamp test (a warp-uniform choice per record).
constexpr float kClampGuard = 0.9989f;

// One contribution of splat r (sweep position jpos) to pixel p of the reverse sweep
// (render.hpp:554-589): steps the pixel's reverse state and accumulates 9 per-lane sums
//   v[0..2] = sum alpha*T*g_rgb                      (rgb gradient)
//   v[3]    = sum t,  t = weight * d_alpha (0 when the 0.999 clamp is active)   (alpha_base gradient)
//   v[4..8] = sum t*dx^2, t*dy^2, t*dx*dy, t*dx, t*dy
// from which the per-record combine (sweep_combine) forms the mean2d and cov gradients:
// dq_i = alpha * d_alpha * (-0.5/det) = ab * nh * t, and the reference's per-contribution terms
// dqi * (2b*dy - 2c*dx) ... are linear in these moments with per-splat coefficients (sum t*q too:
// q is the conic's quadratic form in dx, dy). The arithmetic runs on fast math with explicit FMAs
// (tolerance-checked). CLAMP: the record may reach the 0.999 clamp — the decision,
// which selects the reference's branch (render.hpp:560-573), is recomputed with the forward's exact
// arithmetic whenever the fast alpha is within 1e-4 of the threshold, so both passes always take the
// same branch. Predicated: a lane whose pixel is outside the record's box (or past its last index)
// adds exact zeros and keeps its state.
//
// GSS_BWD_XFACT: a lane's 4 pixels share their column, so dx is per (record, lane): the quadratic
// form is evaluated as q = dy * (ic*dy + ibm2*dx) + ia*dx^2 (2 FMAs per pixel on the lane's
// per-record ax = ia*dx^2, bx = ibm2*dx) and the moments with a dx factor are formed once per record
// from the lane's sums (sum t*dx^2 = dx^2 * sum t, sum t*dx = dx * sum t, sum t*dx*dy = dx * sum t*dy):
// per pixel only sum t, sum t*dy, sum t*dy^2 are swept (bwd_finish_lane completes v[4], v[6], v[7]).
#ifndef GSS_BWD_XFACT
#define GSS_BWD_XFACT 1
#endif
// GSS_BWD_DYINC: the lane's pixel rows are cy0 + 2h, so dy of pixel h is dy0 + 2h (one add per pixel
// instead of re-deriving cy from the row index under register pressure).
#ifndef GSS_BWD_DYINC
#define GSS_BWD_DYINC 1
#endif
#ifndef GSS_BWD_WSEL
#define GSS_BWD_WSEL 1
#endif
struct BwdLane {
  float dx, ax, bx, dy0;
};
__device__ __forceinline__ BwdLane bwd_lane(const SplatRec& r, const BwdConic& k, const PixB& p0) {
  const float dx = p0.cx - r.mx;
#if GSS_BWD_KFOLD
  return BwdLane{dx, k.sia * (dx * dx), k.sibm2 * dx, p0.cy - r.my};
#else
  return BwdLane{dx, k.ia * (dx * dx), k.ibm2 * dx, p0.cy - r.my};
#endif
}
__device__ __forceinline__ void bwd_finish_lane(const BwdLane& l, float v[9]) {
#if GSS_BWD_XFACT
  v[4] = (l.dx * l.dx) * v[3];
  v[6] = l.dx * v[8];
  v[7] = l.dx * v[3];
#endif
}
template <bool CLAMP, int H>
__device__ __forceinline__ bool bwd_contrib(const SplatRec& r, const BwdConic& k, const BwdLane& l, bool xin,
                                            int jpos, PixB& p, float v[9]) {
  const bool ok = xin & (jpos < p.L) & (p.y >= r.by0) & (p.y < r.by1);
#if GSS_BWD_XFACT
  const float dx = l.dx, dy = (GSS_BWD_DYINC && H > 0) ? l.dy0 + (float)(2 * H) : (H == 0 ? l.dy0 : p.cy - r.my);
#if GSS_BWD_KFOLD
  float q = __fmaf_rn(dy, __fmaf_rn(k.sic, dy, l.bx), l.ax);  // kExpHalf * the quadratic form
#else
  float q = __fmaf_rn(dy, __fmaf_rn(k.ic, dy, l.bx), l.ax);
#endif
#else
  const float dx = p.cx - r.mx, dy = p.cy - r.my;
  const float dxx = dx * dx, dyy = dy * dy, dxy = dx * dy;
  float q = __fmaf_rn(k.ia, dxx, __fmaf_rn(k.ic, dyy, k.ibm2 * dxy));
#endif
#if GSS_BWD_WSEL
  if constexpr (!CLAMP) {
    // One select per pixel: an idle lane takes weight = +0, so alpha = +0, rcp(1 - 0) = 1 exactly
    // (MUFU.RCP(1) == 1, tools/mufucheck.cu), Tb = T, S unchanged and t = +-0 — the partials of
    // the three-select form below, bit for bit (x + -0 == x).
#if GSS_BWD_XFACT && GSS_BWD_KFOLD
    const float weight = ok ? ex2_fast(fminf(q, 0.0f)) : 0.0f;
#else
    const float weight = ok ? ex2_fast(kExpHalf * fmaxf(q, 0.0f)) : 0.0f;
#endif
    const float alpha = r.ab * weight;
    const float inv1m = rcp_fast(1.0f - alpha);
    const float Tb = p.T * inv1m;
    const float w_rgb = alpha * Tb;
    v[0] = __fmaf_rn(w_rgb, p.g0, v[0]);
    v[1] = __fmaf_rn(w_rgb, p.g1, v[1]);
    v[2] = __fmaf_rn(w_rgb, p.g2, v[2]);
    const float dot_c = __fmaf_rn(r.r, p.g0, __fmaf_rn(r.g, p.g1, r.bl * p.g2));
    const float d_alpha = __fmaf_rn(Tb, dot_c, -p.S * inv1m);
    p.S = __fmaf_rn(dot_c, w_rgb, p.S);
    p.T = Tb;
    const float t = weight * d_alpha;
    v[3] += t;
#if GSS_BWD_XFACT
    const float tdy = t * dy;
    v[8] += tdy;
    v[5] = __fmaf_rn(tdy, dy, v[5]);
    (void)dx;
#else
    v[4] = __fmaf_rn(t, dxx, v[4]);
    v[5] = __fmaf_rn(t, dyy, v[5]);
    v[6] = __fmaf_rn(t, dxy, v[6]);
    v[7] = __fmaf_rn(t, dx, v[7]);
    v[8] = __fmaf_rn(t, dy, v[8]);
#endif
    return ok;
  }
#endif
#if GSS_BWD_XFACT && GSS_BWD_KFOLD
  q = (q > 0.0f || !ok) ? 0.0f : q;  // scaled form: an idle lane evaluates at 0
  const float weight = ex2_fast(q);  // exp(-q/2)
#else
  q = (q < 0.0f || !ok) ? 0.0f : q;  // an idle lane evaluates at q = 0: every term stays finite
  const float weight = ex2_fast(kExpHalf * q);  // exp(-q/2)
#endif
  bool clamped = false;
  float alpha;
  if (CLAMP) {
    float raw = r.ab * weight;
    const bool near = ok && fabsf(raw - 0.999f) < 1e-4f;
    if (__any_sync(0xffffffffu, near)) {
      if (near) raw = contrib_eval(r, p.cx, p.cy).clamped ? 1.0f : 0.0f;
    }
    clamped = raw > 0.999f;
    alpha = ok ? (clamped ? 0.999f : r.ab * weight) : 0.0f;
  } else {
    alpha = ok ? r.ab * weight : 0.0f;
  }
  const float inv1m = rcp_fast(1.0f - alpha);
  const float Tb = ok ? p.T * inv1m : p.T;  // transmittance before this contribution
  const float w_rgb = alpha * Tb;
  v[0] = __fmaf_rn(w_rgb, p.g0, v[0]);
  v[1] = __fmaf_rn(w_rgb, p.g1, v[1]);
  v[2] = __fmaf_rn(w_rgb, p.g2, v[2]);
  const float dot_c = __fmaf_rn(r.r, p.g0, __fmaf_rn(r.g, p.g1, r.bl * p.g2));
  const float d_alpha = __fmaf_rn(Tb, dot_c, -p.S * inv1m);
  p.S = __fmaf_rn(dot_c, w_rgb, p.S);
  p.T = Tb;
  const float t = (ok && !clamped) ? weight * d_alpha : 0.0f;  // render.hpp:572-586 only when not clamped
  v[3] += t;
#if GSS_BWD_XFACT
  const float tdy = t * dy;
  v[8] += tdy;
  v[5] = __fmaf_rn(tdy, dy, v[5]);
  (void)dx;
#else
  v[4] = __fmaf_rn(t, dxx, v[4]);
  v[5] = __fmaf_rn(t, dyy, v[5]);
  v[6] = __fmaf_rn(t, dxy, v[6]);
  v[7] = __fmaf_rn(t, dx, v[7]);
  v[8] = __fmaf_rn(t, dy, v[8]);
#endif
  return ok;
}

// The lane's pixels of one record, unrolled with the pixel index as a template argument (row h of
// the lane is cy0 + 2h); returns how many contributed.
template <bool CLAMP, int H = 0>
__device__ __forceinline__ int bwd_pixels(const SplatRec& r, const BwdConic& k, const BwdLane& l, bool xin, int jpos,
                                          PixB* px, float v[9]) {
  if constexpr (H < GSS_BWD_PPT) {
    const int u = bwd_contrib<CLAMP, H>(r, k, l, xin, jpos, px[H], v) ? 1 : 0;
    return u + bwd_pixels<CLAMP, H + 1>(r, k, l, xin, jpos, px, v);
  } else {
    return 0;
  }
}

// The 9 SlotAcc terms (rgb3, mean2d2, cov3, alpha_base; render.hpp:538) of one record from its 9
// swept sums (bwd_contrib): with f = ab * (-0.5/det) and Sq = ia*Sxx + ic*Syy + ibm2*Sxy,
//   mean2d = f * (2b*Sy - 2c*Sx, 2b*Sx - 2a*Sy),  cov = f * (Syy - c*Sq, 2b*Sq - 2*Sxy, Sxx - a*Sq).
__device__ __forceinline__ void sweep_combine(const SplatRec& r, const BwdConic& k, const float u[9], float o[9]) {
  const float f = r.ab * k.nh, b2 = 2.0f * r.b;
  const float sq = __fmaf_rn(k.ia, u[4], __fmaf_rn(k.ic, u[5], k.ibm2 * u[6]));
  o[0] = u[0];
  o[1] = u[1];
  o[2] = u[2];
  o[3] = f * __fmaf_rn(b2, u[8], -2.0f * r.c * u[7]);
  o[4] = f * __fmaf_rn(b2, u[7], -2.0f * r.a * u[8]);
  o[5] = f * __fmaf_rn(-r.c, sq, u[5]);
  o[6] = f * __fmaf_rn(b2, sq, -2.0f * u[6]);
  o[7] = f * __fmaf_rn(-r.a, sq, u[4]);
  o[8] = u[3];
}

// Warp reduce-scatter of 9 values in 12 shuffles (9 x 5 butterflies would take 45; padding to 16
// takes 16): the value set is halved per lane bit with minimal padding, 9 -> 5 -> 3 -> 2 -> 1
// (bits 4, 3, 2, 1), then lanes 2k and 2k+1 add. Afterwards lane l holds the warp total of value
// index reduce_scatter_index(l) (-1: a padding slot). Fixed order: deterministic.
__device__ __forceinline__ int reduce_scatter_index(int lane) {
  const int j3 = ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);  // of the 3-set (3 = padding)
  const int j5 = ((lane >> 3) & 1) * 3 + j3;                   // of the 5-set (5.. = padding)
  const int j10 = ((lane >> 4) & 1) * 5 + j5;                  // of the 10 slots (9 = padding)
  return (j3 < 3 && j5 < 5 && j10 < 9) ? j10 : -1;
}
__device__ __forceinline__ float warp_reduce_scatter9(const float v[9], int lane) {
  float x[5];
  {  // bit 4: 9 values (+1 padding) -> 5
    const bool up = (lane & 16) != 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const float lo = v[i], hi = i + 5 < 9 ? v[i + 5] : 0.0f;
      x[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, 16);
    }
  }
  float y[3];
  {  // bit 3: 5 values (+1 padding) -> 3
    const bool up = (lane & 8) != 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const float lo = x[i], hi = i + 3 < 5 ? x[i + 3] : 0.0f;
      y[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, 8);
    }
  }
  float z[2];
  {  // bit 2: 3 values (+1 padding) -> 2
    const bool up = (lane & 4) != 0;
    const float hi1 = 0.0f;
    z[0] = (up ? y[2] : y[0]) + __shfl_xor_sync(0xffffffffu, up ? y[0] : y[2], 4);
    z[1] = (up ? hi1 : y[1]) + __shfl_xor_sync(0xffffffffu, up ? y[1] : hi1, 4);
  }
  const bool up = (lane & 2) != 0;  // bit 1: 2 values -> 1
  const float u = (up ? z[1] : z[0]) + __shfl_xor_sync(0xffffffffu, up ? z[0] : z[1], 2);
  return u + __shfl_xor_sync(0xffffffffu, u, 1);
}

// Reverse sweep (render.hpp:542-589) per 16x16 tile: 64 threads, 4 pixels each (rows ly, ly + 2,
// ly + 4, ly + 6 of an 8-row warp band), so a splat's 9 gradient terms are pre-summed per lane
// over 4 pixels (predicated, interleavable) and reduced once per warp. Per batch, each warp ballots which records can reach its band (pixel
// box intersects the band and sweep position < the band's largest last-contribution index) and
// walks only those. One partial SlotAcc per (splat, tile) instance, fixed-order sums (no float
// atomics, deterministic). partial layout: [instance][9] = rgb3, m2d2, cov3, ab.
constexpr int kBwdPPT = GSS_BWD_PPT;              // pixels per thread
constexpr int kBwdThreads = kTilePix / kBwdPPT;
constexpr int kBwdWarps = kBwdThreads / 32;
constexpr int kBand = 2 * kBwdPPT;                // rows per warp band
__global__ void GSS_BWD_BOUNDS backward_kernel(const SplatRec* __restrict__ recs,
                                                               const int32_t* __restrict__ vals,
                                                               const int2* __restrict__ ranges,
                                                               const int32_t* __restrict__ tile_order, Win w, float bg0,
                                                               float bg1, float bg2, const float* __restrict__ fT_in,
                                                               const int32_t* __restrict__ last_in,
                                                               const float* __restrict__ d_img, float* partials) {
  static_assert(kBwdBatch % 64 == 0, "whole 64-bit record masks per warp");
  __shared__ SplatRec sh[kBwdBatch];
  __shared__ BwdConic shk[kBwdBatch];
  __shared__ int32_t sinst[kBwdBatch];  // the record's (splat, this tile) instance index
  constexpr int kNv = 9;  // swept sums per record (bwd_contrib)
  __shared__ float red[kBwdBatch][kBwdWarps][kNv];
  __shared__ unsigned long long wmask[kBwdWarps][kBwdMasks];
  __shared__ int smax;
  const int tile = tile_of(tile_order);
  const int tx = tile % w.tw, ty = tile / w.tw;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lx = lane & 15, ly = warp * kBand + (lane >> 4);
  const int2 rg = ranges[tile];
  const int bx0w = w.px0 + tx * kTileSize, by0w = w.py0 + ty * kTileSize + warp * kBand;  // warp band origin
  PixB px[kBwdPPT];
  int lmax = 0;
#pragma unroll
  for (int h = 0; h < kBwdPPT; ++h) {
    PixB& p = px[h];
    p.x = w.px0 + tx * kTileSize + lx;
    p.y = w.py0 + ty * kTileSize + ly + 2 * h;
    p.cx = (float)p.x + 0.5f;
    p.cy = (float)p.y + 0.5f;
    p.L = 0;
    p.T = 1.0f;
    p.g0 = p.g1 = p.g2 = 0.0f;
    if (p.x < w.px0 + w.pw && p.y < w.py0 + w.ph) {
      const int64_t pix = (int64_t)(p.y - w.py0) * w.pw + (p.x - w.px0);
      p.L = last_in[pix];
      p.T = fT_in[pix];
      p.g0 = d_img[pix * 3];
      p.g1 = d_img[pix * 3 + 1];
      p.g2 = d_img[pix * 3 + 2];
      if (p.g0 == 0.0f && p.g1 == 0.0f && p.g2 == 0.0f) p.L = 0;  // render.hpp:551
    }
    p.S = __fmaf_rn(p.T * bg0, p.g0, __fmaf_rn(p.T * bg1, p.g1, (p.T * bg2) * p.g2));  // (final_T * bg) . g
    lmax = max(lmax, p.L);
  }
  if (threadIdx.x == 0) smax = 0;
  const int wl = __reduce_max_sync(0xffffffffu, lmax);  // the band's largest last index
  __syncthreads();
  if (lane == 0 && wl > 0) atomicMax(&smax, wl);
  __syncthreads();
  const int Lmax = smax;
  const int vidx = reduce_scatter_index(lane);
#if GSS_RASTER_STATS
  unsigned long long st_walk = 0, st_use = 0;
#endif
  for (int bend = Lmax; bend > 0; bend -= kBwdBatch) {
    const int bstart = max(0, bend - kBwdBatch);
    const int nb = bend - bstart;
    __syncthreads();
    for (int j = threadIdx.x; j < nb; j += kBwdThreads) {
      load_rec(&sh[j], recs, vals[rg.x + bstart + j]);
      const SplatRec& r = sh[j];
      const float inv = 1.0f / r.det;  // det > 0 for every binned splat
#if GSS_BWD_KFOLD
      {
        const float ia = r.c * inv, ibm2 = -2.0f * (r.b * inv), ic = r.a * inv;
        shk[j] = BwdConic{ia, ibm2, ic, -0.5f * inv, kExpHalf * ia, kExpHalf * ibm2, kExpHalf * ic, 0.0f};
      }
#else
      shk[j] = BwdConic{r.c * inv, -2.0f * (r.b * inv), r.a * inv, -0.5f * inv};
#endif
      int tx0, ty0, ntx, nty;
      tile_box(r, w, tx0, ty0, ntx, nty);
      sinst[j] = r.off + (ty - ty0) * ntx + (tx - tx0);
    }
    __syncthreads();
    unsigned long long mk[kBwdMasks];
#pragma unroll
    for (int h = 0; h < kBwdBatch / 32; ++h) {
      const int jl = h * 32 + lane;
      bool hit = false;
      if (jl < nb && bstart + jl < wl) {
        const int4 bx = *reinterpret_cast<const int4*>(&sh[jl].bx0);
        hit = bx.x <= bx0w + 15 && bx.y > bx0w && bx.z <= by0w + kBand - 1 && bx.w > by0w;
      }
      const unsigned long long bal = (unsigned long long)__ballot_sync(0xffffffffu, hit) << (32 * (h & 1));
      mk[h >> 1] = (h & 1) ? (mk[h >> 1] | bal) : bal;
    }
    if (lane == 0) {
#pragma unroll
      for (int h = 0; h < kBwdMasks; ++h) wmask[warp][h] = mk[h];
    }
#if GSS_BWD_BATCH == 64
    // One 64-record batch walked as two 32-bit halves (32-bit find-last-set on the uniform
    // datapath instead of 64-bit arithmetic per record): high half first, back to front.
    {
      const unsigned ml = (unsigned)mk[0];
      unsigned m = (unsigned)(mk[0] >> 32);
      int hb = 32;
      if (m == 0) {
        m = ml;
        hb = 0;
      }
      while (m) {
        const int bit = 31 - __clz(m);
        const int jj = hb + bit;
        m ^= 1u << bit;
        if (m == 0 && hb == 32) {
          m = ml;
          hb = 0;
        }
#else
#pragma unroll
    for (int h = kBwdMasks - 1; h >= 0; --h) {
      for (unsigned long long m = mk[h]; m;) {
        const int jj = h * 64 + 63 - __clzll(m);  // reverse order: back to front
        m &= ~(1ull << (jj & 63));
#endif
        const SplatRec r = sh[jj];
        const BwdConic k = shk[jj];
        const bool xin = (px[0].x >= r.bx0) & (px[0].x < r.bx1);
        const BwdLane bl = bwd_lane(r, k, px[0]);
        float v[kNv];
#pragma unroll
        for (int i = 0; i < kNv; ++i) v[i] = 0.0f;
#if GSS_RASTER_STATS
        ++st_walk;
#endif
        const int nuse = r.ab > kClampGuard ? bwd_pixels<true>(r, k, bl, xin, bstart + jj, px, v)
                                            : bwd_pixels<false>(r, k, bl, xin, bstart + jj, px, v);
#if GSS_RASTER_STATS
        st_use += nuse;
#endif
        (void)nuse;
        bwd_finish_lane(bl, v);
        // A record no lane contributed to reduces exact zeros: the same partial without a vote.
        const float tot = warp_reduce_scatter9(v, lane);
        if ((lane & 1) == 0 && vidx >= 0) red[jj][warp][vidx] = tot;
      }
    }
    __syncthreads();
    // Fixed-order cross-warp sum over the warps that walked the record, then the record's 9 SlotAcc
    // terms: one instance partial per splat of the batch (a thread per record).
    for (int jj = threadIdx.x; jj < nb; jj += kBwdThreads) {
      float u[kNv];
#pragma unroll
      for (int i = 0; i < kNv; ++i) u[i] = 0.0f;
#pragma unroll
      for (int q = 0; q < kBwdWarps; ++q)
        if ((wmask[q][jj >> 6] >> (jj & 63)) & 1ull)
#pragma unroll
          for (int i = 0; i < kNv; ++i) u[i] += red[jj][q][i];
      float o[9];
      sweep_combine(sh[jj], shk[jj], u, o);
      float* dst = partials + (int64_t)sinst[jj] * 9;
#pragma unroll
      for (int i = 0; i < 9; ++i) dst[i] = o[i];
    }
  }
  // Records behind every pixel's last contribution (sweep position >= Lmax: the T-stop tail) get
  // exact-zero partials here, so the partials buffer needs no clearing pass before the sweep.
  for (int j = Lmax + threadIdx.x; j < rg.y - rg.x; j += kBwdThreads) {
    const SplatRec& r = recs[vals[rg.x + j]];
    int tx0, ty0, ntx, nty;
    tile_box(r, w, tx0, ty0, ntx, nty);
    float* dst = partials + (int64_t)(r.off + (ty - ty0) * ntx + (tx - tx0)) * 9;
#pragma unroll
    for (int i = 0; i < 9; ++i) dst[i] = 0.0f;
  }
#if GSS_RASTER_STATS
  if (lane == 0) {
    atomicAdd(&g_rstats[5], st_walk);
    atomicAdd(&g_rstats[6], st_walk * 32ull * kBwdPPT);
  }
  atomicAdd(&g_rstats[7], st_use);
#endif
}

// Per-slot sums of the instance partials in depth order: a warp owns 32 consecutive depth
// positions, whose instance ranges [offsets[i], offsets[i+1]) are adjacent — one contiguous span.
// The span is staged into SMEM in chunks of kSumChunk instances with every 4-byte piece in flight
// (LDGSTS, coalesced), and each lane adds its own slot's instances from SMEM in instance order
// (fixed order: deterministic). The sum lands at the slot the sort payload names.
constexpr int kSumWarps = 8;
constexpr int kSumChunk = 128;  // instances per staged chunk (4.5 KB per warp)
__global__ void __launch_bounds__(kSumWarps * 32) slot_sum_depth_kernel(int64_t V, const int32_t* __restrict__ offsets,
                                                                      const uint64_t* __restrict__ pay,
                                                                      const float* __restrict__ partials, float* sums) {
  __shared__ __align__(16) float stage[kSumWarps][kSumChunk * 9];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i0 = ((int64_t)blockIdx.x * kSumWarps + warp) * 32;
  if (i0 >= V) return;
  const int64_t i = i0 + lane;
  const bool valid = i < V;
  const int64_t iend = i0 + 32 < V ? i0 + 32 : V;
  const int32_t o0 = valid ? offsets[i] : offsets[iend];
  const int32_t o1 = valid ? offsets[i + 1] : o0;
  const int32_t s0 = __shfl_sync(0xffffffffu, o0, 0);
  const int32_t s1 = offsets[iend];
  float acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0f;
  float* st = stage[warp];
  // chunks start on multiples of 4 instances (36 x 4 = 144 bytes: 16-byte aligned), so the span is
  // copied in 16-byte pieces (the instances before s0 are copied and ignored)
  for (int32_t c0 = s0 & ~3; c0 < s1; c0 += kSumChunk) {
    const int n = (s1 - c0 < kSumChunk ? s1 - c0 : kSumChunk) * 9;
    const float* src = partials + (int64_t)c0 * 9;
    __syncwarp();
    const int n4 = n >> 2;
    for (int e = lane; e < n4; e += 32) cp_async16(st + 4 * e, src + 4 * e);
    for (int e = 4 * n4 + lane; e < n; e += 32) cp_async4(st + e, src + e);
    cp_async_wait_all();
    __syncwarp();
    const int32_t a = o0 > c0 ? o0 : c0, b = o1 < c0 + kSumChunk ? o1 : c0 + kSumChunk;
    for (int32_t j = a; j < b; ++j) {
      const float* q = st + (j - c0) * 9;
#pragma unroll
      for (int c = 0; c < 9; ++c) acc[c] += q[c];
    }
  }
  if (valid) {
    const int64_t k = (int64_t)(uint32_t)pay[i];
#pragma unroll
    for (int c = 0; c < 9; ++c) sums[k * 9 + c] = acc[c];
  }
}

// Per-slot sums in depth order as a warp-wide segmented scan (GSS_SUM_SEG): the warp's 32 slots own
// one contiguous instance span, which the warp walks 32 instances at a time (lane = instance, the 9
// values loaded coalesced); a segmented inclusive scan (heads = the slots' first instances) sums
// each slot's piece of the chunk in a fixed tree order, and the piece's last lane adds it to the
// slot's accumulator in SMEM (pieces in chunk order). Every lane does useful work whatever the
// slots' instance counts — the lane-per-slot loop above waits for the warp's largest splat.
// Deterministic (fixed order); the order differs from the lane-per-slot loop's by rounding only.
#ifndef GSS_SUM_SEG
#define GSS_SUM_SEG 1
#endif
#ifndef GSS_SUM_U
#define GSS_SUM_U 4
#endif
__global__ void __launch_bounds__(kSumWarps * 32) slot_sum_seg_kernel(int64_t V, const int32_t* __restrict__ offsets,
                                                                    const uint64_t* __restrict__ pay,
                                                                    const float* __restrict__ partials, float* sums) {
  __shared__ float acc[kSumWarps][32][9];
  __shared__ int8_t owner_at[kSumWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i0 = ((int64_t)blockIdx.x * kSumWarps + warp) * 32;
  if (i0 >= V) return;
  const int64_t i = i0 + lane;
  const bool valid = i < V;
  const int64_t iend = i0 + 32 < V ? i0 + 32 : V;
  const int32_t o0 = valid ? offsets[i] : offsets[iend];
  const int32_t o1 = valid ? offsets[i + 1] : o0;
  const int32_t s0 = __shfl_sync(0xffffffffu, o0, 0);
  const int32_t s1 = offsets[iend];
  float* A = acc[warp][lane];
#pragma unroll
  for (int c = 0; c < 9; ++c) A[c] = 0.0f;
  __syncwarp();
  // GSS_SUM_U chunks' loads in flight before their scans: a warp whose slots include a splat with
  // thousands of tile instances walks a long span, and that warp's serial chain of load latencies
  // is the kernel's tail.
  for (int32_t cg = s0; cg < s1; cg += 32 * GSS_SUM_U) {
    float xs[GSS_SUM_U][9];
#pragma unroll
    for (int u = 0; u < GSS_SUM_U; ++u) {
      const int32_t j = cg + 32 * u + lane;
      const bool in = j < s1;
      const float* src = partials + (int64_t)j * 9;
#pragma unroll
      for (int c = 0; c < 9; ++c) xs[u][c] = in ? __ldg(src + c) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < GSS_SUM_U; ++u) {
    const int32_t cb = cg + 32 * u;
    if (cb >= s1) break;
    const bool head = valid && o1 > o0 && o0 >= cb && o0 < cb + 32;
    if (head) owner_at[warp][o0 - cb] = (int8_t)lane;
    const unsigned hmask = __reduce_or_sync(0xffffffffu, head ? 1u << (o0 - cb) : 0u);
    const unsigned open = __ballot_sync(0xffffffffu, valid && o0 <= cb && cb < o1);  // the slot open at cb
    __syncwarp();
    const int32_t j = cb + lane;
    const bool in = j < s1;
    float* x = xs[u];
    const unsigned below = hmask & (0xffffffffu >> (31 - lane));  // heads at lanes 0..lane
    const int hp = below ? 31 - __clz(below) : -1;                // -1: the piece continues a slot
    const int lim = hp >= 0 ? lane - hp : lane;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        const float y = __shfl_up_sync(0xffffffffu, x[c], d);
        if (d <= lim) x[c] += y;
      }
    }
    const bool end = in && (lane == 31 || j + 1 == s1 || ((hmask >> (lane + 1)) & 1u));
    if (end) {
      const int t = hp >= 0 ? owner_at[warp][hp] : __ffs(open) - 1;
      float* T = acc[warp][t];
#pragma unroll
      for (int c = 0; c < 9; ++c) T[c] += x[c];
    }
    __syncwarp();
    }
  }
  if (valid) {
    const int64_t k = (int64_t)(uint32_t)pay[i];
#pragma unroll
    for (int c = 0; c < 9; ++c) sums[k * 9 + c] = A[c];
  }
}

// render.hpp:600-638 + project_geo_backward (render.hpp:152-237), per slot.
// Per-slot sums of the backward's instance partials (CSR by slot: instances of slot k are
// [offsets[k], offsets[k+1])), in a fixed order: each lane sums its own slot's first kHead
// instances sequentially (2x unrolled so loads overlap), then the warp sums the tails of big
// splats (near-camera Gaussians cover hundreds of tiles) cooperatively, 4x unrolled, with a
// fixed butterfly. Light on registers, so many warps hide the load latency.
constexpr int kSumThreads = 256;
__global__ void __launch_bounds__(kSumThreads) slot_sum_kernel(int64_t V, const int32_t* slot_off,
                                                               const int32_t* ntiles,
                                                               const float* __restrict__ partials, float* sums) {
  constexpr int kHead = 32;
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * kSumThreads + threadIdx.x;
  const int64_t kw = k - lane;
  if (kw >= V) return;
  int32_t o0 = 0, o1 = 0;
  if (k < V) {
    o0 = slot_off[k];
    o1 = o0 + ntiles[k];
  }
  float acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0f;
  const int32_t hend = min(o1, o0 + kHead);
  int32_t i = o0;
  for (; i + 3 < hend; i += 4) {  // 36 loads in flight, summed in instance order
    float a[4][9];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < 9; ++c) a[u][c] = partials[(int64_t)(i + u) * 9 + c];
#pragma unroll
    for (int c = 0; c < 9; ++c) acc[c] = (((acc[c] + a[0][c]) + a[1][c]) + a[2][c]) + a[3][c];
  }
  for (; i < hend; ++i)
#pragma unroll
    for (int c = 0; c < 9; ++c) acc[c] += partials[(int64_t)i * 9 + c];
  unsigned big = __ballot_sync(0xffffffffu, o1 - o0 > kHead);
  while (big) {
    const int b = __ffs(big) - 1;
    big &= big - 1;
    const int32_t t0 = __shfl_sync(0xffffffffu, o0, b) + kHead, t1 = __shfl_sync(0xffffffffu, o1, b);
    float tail[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) tail[c] = 0.0f;
    int32_t j = t0 + lane;
    for (; j + 96 < t1; j += 128) {
      float x[4][9];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 9; ++c) x[u][c] = partials[(int64_t)(j + 32 * u) * 9 + c];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 9; ++c) tail[c] += x[u][c];
    }
    for (; j < t1; j += 32)
#pragma unroll
      for (int c = 0; c < 9; ++c) tail[c] += partials[(int64_t)j * 9 + c];
#pragma unroll
    for (int c = 0; c < 9; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tail[c] += __shfl_xor_sync(0xffffffffu, tail[c], o);
      if (lane == b) acc[c] += tail[c];
    }
  }
  if (k < V)
#pragma unroll
    for (int c = 0; c < 9; ++c) sums[k * 9 + c] = acc[c];
}

constexpr int kChainThreads = 128;
#ifndef GSS_CHAIN_MINB
#define GSS_CHAIN_MINB 6  // 6 blocks of 128 threads per SM (80 registers): the chain is latency bound
#endif
constexpr int kChainRow = 49;     // odd row pitch: conflict-free per-lane row access
// Warp-cooperative: a warp owns 32 consecutive slots. It sums each slot's instance partials with
// all lanes, stages the slots' 49-float non-geometric rows in SMEM with coalesced loads; each lane
// then runs the reference chain for its slot, and the 59 outputs are written back through SMEM
// with coalesced stores.
template <int DEG>
__global__ void __launch_bounds__(kChainThreads, GSS_CHAIN_MINB) chain_kernel(SceneDev s, Cam cam, Win w, int64_t V,
                                                              const SplatRec* recs, const float* sums,
                                                              float* gg, int64_t gstride,
                                                              float* gn, int64_t nstride, float* mean2d) {
  __shared__ float row_s[kChainThreads / 32][32][kChainRow];
  __shared__ float geo_s[kChainThreads / 32][32][11];  // the 10 geometric gradients, odd pitch
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t k0 = (int64_t)blockIdx.x * kChainThreads + warp * 32;
  if (k0 >= V) return;
  const int nk = (V - k0) < 32 ? (int)(V - k0) : 32;
  float(*rows)[kChainRow] = row_s[warp];
  stage_rows<kChainRow>(s, k0, nk, 49, lane, rows);
  const int64_t k = k0 + lane;
  // Geometric gradients (row columns 0..9) live in registers; the 49 non-geometric ones overwrite
  // this lane's staged non-geometric row in place (column 10 + i -> slot i, each slot read before
  // it is written), which keeps the kernel's register footprint small enough for occupancy.
  float out[10];
#pragma unroll
  for (int i = 0; i < 10; ++i) out[i] = 0.0f;
  float* orow = rows[lane];
  float sa[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) sa[i] = lane < nk ? sums[(k0 + lane) * 9 + i] : 0.0f;
  const int id = lane < nk ? s.ids[k] : 0;
  const float* g = s.geo + (int64_t)id * s.geo_stride;
  Proj p;
  f3 t;
  const bool valid = lane < nk && project_geo(cam, g, s.lp, p, t);
  if (valid) {
    const SplatRec r = recs[k];
    const float* ng = rows[lane];
    const float ab = r.ab;
    const float d_opacity = 0.0f + sa[8] * ab * (1.0f - ab);
    const f3 cp = cam_position(cam);
    const f3 dir{g[0] - cp.x, g[1] - cp.y, g[2] - cp.z};
    const float dn = sqrtf(dir.x * dir.x + dir.y * dir.y + dir.z * dir.z);
    f3 dmd{0.0f, 0.0f, 0.0f};
    if (dn > 1e-12f) {
      const float inv = 1.0f / dn;
      const f3 u{dir.x * inv, dir.y * inv, dir.z * inv};
      float basis[16];
      f3 bgr[16];
      sh_basis(u.x, u.y, u.z, DEG, basis);
      sh_basis_grad(u.x, u.y, u.z, DEG, bgr);
      constexpr int nb = (DEG + 1) * (DEG + 1);
      float gc[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {  // eval_sh_clamp_mask (sh.hpp:114-125)
        float v = 0.5f;
#pragma unroll
        for (int b = 0; b < nb; ++b) v += basis[b] * ng[1 + 3 * b + c];
        gc[c] = (v < 0.0f || v > 1.0f) ? 0.0f : sa[c];
      }
      f3 ddir{0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int b = 0; b < nb; ++b) {  // eval_sh_backward (sh.hpp:92-110)
        float coef_dot = 0.0f;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          coef_dot += ng[1 + 3 * b + c] * gc[c];
          orow[1 + 3 * b + c] = 0.0f + basis[b] * gc[c];
        }
        ddir.x += bgr[b].x * coef_dot;
        ddir.y += bgr[b].y * coef_dot;
        ddir.z += bgr[b].z * coef_dot;
      }
      const float dotp = u.x * ddir.x + u.y * ddir.y + u.z * ddir.z;
      const float inv2 = 1.0f / dn;
      dmd = f3{(ddir.x - u.x * dotp) * inv2, (ddir.y - u.y * dotp) * inv2, (ddir.z - u.z * dotp) * inv2};
#pragma unroll
      for (int i = 1 + 3 * nb; i < 49; ++i) orow[i] = 0.0f;  // bands above DEG
    } else {
#pragma unroll
      for (int i = 1; i < 49; ++i) orow[i] = 0.0f;
    }
    orow[0] = d_opacity;
    out[0] += dmd.x;
    out[1] += dmd.y;
    out[2] += dmd.z;
    // project_geo_backward
    const float dmx = sa[3], dmy = sa[4], da = sa[5], db = sa[6], dc = sa[7];
    const float iz = 1.0f / t.z, iz2 = iz * iz;
    const float qw = g[6], qx = g[7], qy = g[8], qz = g[9];
    const float qn = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
    const float qinv = qn > 1e-12f ? 1.0f / qn : 0.0f;
    const float uq[4] = {qw * qinv, qx * qinv, qy * qinv, qz * qinv};
    float R[9];
    quat_to_rot(uq[0], uq[1], uq[2], uq[3], R);
    const float es[3] = {gss_expf(g[3]), gss_expf(g[4]), gss_expf(g[5])};
    float B[9], S[9];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      B[i * 3 + 0] = R[i * 3 + 0] * es[0];
      B[i * 3 + 1] = R[i * 3 + 1] * es[1];
      B[i * 3 + 2] = R[i * 3 + 2] * es[2];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        S[i * 3 + j] = B[i * 3] * B[j * 3] + B[i * 3 + 1] * B[j * 3 + 1] + B[i * 3 + 2] * B[j * 3 + 2];
    const float fx = cam.fx, fy = cam.fy;
    const float j00 = fx * iz, j02 = -fx * t.x * iz2;
    const float j11 = fy * iz, j12 = -fy * t.y * iz2;
    const float* W = cam.m;
    const float m0[3] = {j00 * W[0] + j02 * W[6], j00 * W[1] + j02 * W[7], j00 * W[2] + j02 * W[8]};
    const float m1[3] = {j11 * W[3] + j12 * W[6], j11 * W[4] + j12 * W[7], j11 * W[5] + j12 * W[8]};
    float v0[3], v1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      v0[i] = S[i * 3] * m0[0] + S[i * 3 + 1] * m0[1] + S[i * 3 + 2] * m0[2];
      v1[i] = S[i * 3] * m1[0] + S[i * 3 + 1] * m1[1] + S[i * 3 + 2] * m1[2];
    }
    float dm0[3], dm1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      dm0[i] = v0[i] * (2.0f * da) + v1[i] * db;
      dm1[i] = v1[i] * (2.0f * dc) + v0[i] * db;
    }
    float dS[9], dB[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) dS[i * 3 + j] = da * m0[i] * m0[j] + db * m0[i] * m1[j] + dc * m1[i] * m1[j];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float a2 = 0.0f;
#pragma unroll
        for (int q = 0; q < 3; ++q) a2 += (dS[i * 3 + q] + dS[q * 3 + i]) * B[q * 3 + j];
        dB[i * 3 + j] = a2;
      }
    float G[9];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      G[i * 3 + 0] = dB[i * 3 + 0] * es[0];
      G[i * 3 + 1] = dB[i * 3 + 1] * es[1];
      G[i * 3 + 2] = dB[i * 3 + 2] * es[2];
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      float a2 = 0.0f;
#pragma unroll
      for (int i = 0; i < 3; ++i) a2 += dB[i * 3 + j] * R[i * 3 + j];
      out[3 + j] += a2 * es[j];
    }
    const float qw_ = uq[0], qx_ = uq[1], qy_ = uq[2], qz_ = uq[3];
#define GG(i, j) G[(i) * 3 + (j)]
    float dq[4];
    dq[0] = 2.0f * (-qz_ * GG(0, 1) + qy_ * GG(0, 2) + qz_ * GG(1, 0) - qx_ * GG(1, 2) - qy_ * GG(2, 0) +
                    qx_ * GG(2, 1));
    dq[1] = 2.0f * (qy_ * GG(0, 1) + qz_ * GG(0, 2) + qy_ * GG(1, 0) - 2.0f * qx_ * GG(1, 1) - qw_ * GG(1, 2) +
                    qz_ * GG(2, 0) + qw_ * GG(2, 1) - 2.0f * qx_ * GG(2, 2));
    dq[2] = 2.0f * (-2.0f * qy_ * GG(0, 0) + qx_ * GG(0, 1) + qw_ * GG(0, 2) + qx_ * GG(1, 0) + qz_ * GG(1, 2) -
                    qw_ * GG(2, 0) + qz_ * GG(2, 1) - 2.0f * qy_ * GG(2, 2));
    dq[3] = 2.0f * (-2.0f * qz_ * GG(0, 0) - qw_ * GG(0, 1) + qx_ * GG(0, 2) + qw_ * GG(1, 0) -
                    2.0f * qz_ * GG(1, 1) + qy_ * GG(1, 2) + qx_ * GG(2, 0) + qy_ * GG(2, 1));
#undef GG
    const float nq = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);  // quat_normalize_backward
    const float qi = 1.0f / nq;
    const float u4[4] = {qw * qi, qx * qi, qy * qi, qz * qi};
    const float dotq = u4[0] * dq[0] + u4[1] * dq[1] + u4[2] * dq[2] + u4[3] * dq[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) out[6 + i] += (dq[i] - u4[i] * dotq) * qi;
    const float dj00 = dm0[0] * W[0] + dm0[1] * W[1] + dm0[2] * W[2];
    const float dj02 = dm0[0] * W[6] + dm0[1] * W[7] + dm0[2] * W[8];
    const float dj11 = dm1[0] * W[3] + dm1[1] * W[4] + dm1[2] * W[5];
    const float dj12 = dm1[0] * W[6] + dm1[1] * W[7] + dm1[2] * W[8];
    f3 dt;
    dt.x = dmx * fx * iz + dj02 * (-fx * iz2);
    dt.y = dmy * fy * iz + dj12 * (-fy * iz2);
    dt.z = dmx * (-fx * t.x * iz2) + dmy * (-fy * t.y * iz2) + dj00 * (-fx * iz2) + dj11 * (-fy * iz2) +
           dj02 * (2.0f * fx * t.x * iz2 * iz) + dj12 * (2.0f * fy * t.y * iz2 * iz);
    out[0] += W[0] * dt.x + W[3] * dt.y + W[6] * dt.z;
    out[1] += W[1] * dt.x + W[4] * dt.y + W[7] * dt.z;
    out[2] += W[2] * dt.x + W[5] * dt.y + W[8] * dt.z;
  }
  if (lane < nk && !valid) {
#pragma unroll
    for (int i = 0; i < 49; ++i) orow[i] = 0.0f;
  }
  __syncwarp();
  if (lane < nk) {
#pragma unroll
    for (int i = 0; i < 10; ++i) geo_s[warp][lane][i] = out[i];
    if (mean2d) {
      mean2d[k * 2] = sa[3];
      mean2d[k * 2 + 1] = sa[4];
    }
  }
  __syncwarp();
  for (int e = lane; e < nk * 10; e += 32) {
    const int kk = e / 10, c = e - kk * 10;
    gg[(k0 + kk) * gstride + c] = geo_s[warp][kk][c];
  }
  for (int e = lane; e < nk * 49; e += 32) {
    const int kk = e / 49, c = e - kk * 49;
    gn[(k0 + kk) * nstride + c] = rows[kk][c];
  }
}

Win make_window(const gss_viewport& vp) {
  // viewport_pixels (render.hpp:297-304)
  auto cvt = [](double d) -> int {
    if (!(d >= -2147483648.0 && d < 2147483648.0)) return (int)0x80000000u;
    return (int)d;
  };
  int px0 = cvt(std::ceil(double(vp.x0) - 0.5)), px1 = cvt(std::ceil(double(vp.x1) - 0.5));
  int py0 = cvt(std::ceil(double(vp.y0) - 0.5)), py1 = cvt(std::ceil(double(vp.y1) - 0.5));
  px0 = std::max(px0, 0);
  py0 = std::max(py0, 0);
  Win w;
  w.px0 = px0;
  w.py0 = py0;
  w.pw = std::max(0, px1 - px0);
  w.ph = std::max(0, py1 - py0);
  w.tw = (w.pw + kTileSize - 1) / kTileSize;
  w.th = (w.ph + kTileSize - 1) / kTileSize;
  return w;
}

}  // namespace

namespace {

void set_scene(gss_render_ctx* ctx, const gss_render_scene* scene) {
  require(scene->sh_degree >= 0 && scene->sh_degree <= 3, "rasterize_forward: sh_degree must be in [0,3]");
  require(scene->geo_stride >= 10 && scene->nongeo_stride >= 49, "rasterize_forward: bad strides");
  SceneDev& s = ctx->sc;
  s.ids = scene->ids; s.geo = scene->geo; s.geo_stride = scene->geo_stride; s.nongeo = scene->nongeo;
  s.ng_stride = scene->nongeo_stride; s.compact = scene->nongeo_compact; s.slot_map = scene->slot_map;
  s.sh_degree = scene->sh_degree; s.lp = scene->low_pass;
  for (int c = 0; c < 3; ++c) s.bg[c] = scene->background[c];
}

int64_t scene_count(gss_render_ctx* ctx, const gss_render_scene* scene, cudaStream_t st) {
  int64_t V = scene->count;
  if (scene->count_dev) {
    GSS_CUDA(cudaMemcpyAsync(ctx->pinned, scene->count_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GSS_CUDA(cudaStreamSynchronize(st));
    V = ctx->pinned[0];
  }
  require(V >= 0 && V <= INT32_MAX, "rasterize_forward: visible count out of range");
  return V;
}

struct FwdOut {
  float* image;
  const float* gt;
  int gt_width;
  float inv;
  float* d_img;
  float* loss_dev;
  double* loss_sum;
  float* final_T;
  int32_t* ncontrib;
  int64_t* meta;
};

// Everything after the records exist: common to rasterize_forward (records from preprocess) and
// the image-parallel strip forward (records received from other GPUs, re-clipped). Expects
// ctx->recs / ntiles / dkeys_a / order_a filled for V records, boxes clipped to w.
// bin_phase: depth sort, instance offsets, tile keys, tile sort, tile ranges (ctx->I set; the
// sorted instance values end in ctx->vals_a, the ranges in ctx->ranges).
void bin_phase(gss_render_ctx* ctx, const Win& w, int64_t V, cudaStream_t st) {
  const int64_t npix = (int64_t)w.pw * w.ph;
  ctx->I = 0;
  if (npix == 0) return;
  SplatRec* recs = static_cast<SplatRec*>(ctx->recs.p);
  int32_t* nt = static_cast<int32_t*>(ctx->ntiles.p);
  int32_t* offs = static_cast<int32_t*>(ctx->offsets.get((size_t)(V + 1) * 4, st));
  int32_t* soff = static_cast<int32_t*>(ctx->slot_off.get((size_t)std::max<int64_t>(V, 1) * 4, st));
  int64_t I = 0;
  const int ntile = w.tw * w.th;
  int2* ranges = static_cast<int2*>(ctx->ranges.get((size_t)ntile * sizeof(int2), st));
  GSS_CUDA(cudaMemsetAsync(ranges, 0, (size_t)ntile * sizeof(int2), st));
  ctx->vals_a.get(16, st);
  if (V > 0) {
    auto* dka = static_cast<uint32_t*>(ctx->dkeys_a.p);
    auto* dkb = static_cast<uint32_t*>(ctx->dkeys_b.get((size_t)V * 4, st));
    auto* oa = static_cast<uint64_t*>(ctx->order_a.p);
    auto* ob = static_cast<uint64_t*>(ctx->order_b.get((size_t)V * 8, st));
    // 1. stable sort of the V splats by depth (record order breaks ties: ascending id); the payload
    //    carries the slot and its packed tile box.
    cub::DoubleBuffer<uint32_t> ddk(dka, dkb);
    cub::DoubleBuffer<uint64_t> ddv(oa, ob);
    size_t db = 0;
    GSS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, db, ddk, ddv, (int)V, 0, 32, st));
    // 2. instance offsets in depth order; offs[V] = I.
    using CountIt = thrust::transform_iterator<SortedCount, thrust::counting_iterator<int32_t>>;
    size_t tb = 0;
    GSS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, CountIt(thrust::counting_iterator<int32_t>(0),
                                                                    SortedCount{nt, nullptr, (int32_t)V}),
                                           offs, (int)(V + 1), st));
    void* tmp = ctx->cub_tmp.get(std::max(db, tb), st);
    GSS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, db, ddk, ddv, (int)V, 0, 32, st));
    count_launch();
    const uint64_t* order = ddv.Current();
    ctx->pay_sorted = order;
    GSS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, CountIt(thrust::counting_iterator<int32_t>(0),
                                                                SortedCount{nt, order, (int32_t)V}),
                                           offs, (int)(V + 1), st));
    count_launch();
    GSS_CUDA(cudaMemcpyAsync(ctx->pinned + 1, offs + V, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GSS_CUDA(cudaStreamSynchronize(st));
    I = (int64_t)(reinterpret_cast<int32_t*>(ctx->pinned + 1)[0]);
    require(I >= 0 && I <= INT32_MAX, "rasterize_forward: tile instance count overflow");
    auto* ka = static_cast<uint32_t*>(ctx->keys_a.get((size_t)std::max<int64_t>(I, 1) * 4, st));
    auto* kb = static_cast<uint32_t*>(ctx->keys_b.get((size_t)std::max<int64_t>(I, 1) * 4, st));
    auto* va = static_cast<int32_t*>(ctx->vals_a.get((size_t)std::max<int64_t>(I, 1) * 4, st));
    auto* vb = static_cast<int32_t*>(ctx->vals_b.get((size_t)std::max<int64_t>(I, 1) * 4, st));
    duplicate_kernel<<<(unsigned)ceil_div(V, 128), 128, 0, st>>>(recs, order, nt, offs, w, V, ka, va, recs, soff);
    GSS_LAUNCHED();
    if (I > 0) {
      // 3. stable sort of the instances by tile (only the tile bits).
      int tile_bits = 1;
      while ((1ll << tile_bits) < ntile) ++tile_bits;
      cub::DoubleBuffer<uint32_t> dk(ka, kb);
      cub::DoubleBuffer<int32_t> dv(va, vb);
      size_t sb = 0;
      GSS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sb, dk, dv, (int)I, 0, tile_bits, st));
      void* stmp = ctx->cub_tmp.get(std::max(sb, std::max(db, tb)), st);
      GSS_CUDA(cub::DeviceRadixSort::SortPairs(stmp, sb, dk, dv, (int)I, 0, tile_bits, st));
      count_launch();
      // keep the sorted arrays addressable (vals_a) for composite and backward
      if (dk.Current() != ka) std::swap(ctx->keys_a, ctx->keys_b);
      if (dv.Current() != va) std::swap(ctx->vals_a, ctx->vals_b);
      ranges_kernel<<<(unsigned)ceil_div(ceil_div(I, 4), 256), 256, 0, st>>>(static_cast<const uint32_t*>(ctx->keys_a.p), I,
                                                                ranges);
      GSS_LAUNCHED();
    }
  }
  ctx->I = I;
  int32_t* order = static_cast<int32_t*>(ctx->tile_order.get((size_t)ntile * 4, st));
  if (GSS_LPT) {
    tile_order_kernel<<<1, kOrderThreads, 0, st>>>(ranges, ntile, order);
    GSS_LAUNCHED();
  }
}

void ktime_begin(gss_render_ctx* ctx, int kind, cudaStream_t st) {
  if (!ctx->ktiming) return;
  gss_render_ctx::KTime t{kind, nullptr, nullptr};
  for (cudaEvent_t* e : {&t.a, &t.b}) {
    if (!ctx->kfree.empty()) {
      *e = ctx->kfree.back();
      ctx->kfree.pop_back();
    } else {
      GSS_CUDA(cudaEventCreate(e));
    }
  }
  GSS_CUDA(cudaEventRecord(t.a, st));
  ctx->ktimes.push_back(t);
}
void ktime_end(gss_render_ctx* ctx, cudaStream_t st) {
  if (ctx->ktiming) GSS_CUDA(cudaEventRecord(ctx->ktimes.back().b, st));
}

// composite_phase: per-pixel compositing fused with the L1 loss (forward_kernel).
void composite_phase(gss_render_ctx* ctx, const Win& w, int64_t V, const FwdOut& o, cudaStream_t st) {
  const SceneDev& s = ctx->sc;
  const int64_t npix = (int64_t)w.pw * w.ph;
  float* fT = static_cast<float*>(ctx->fT.get((size_t)std::max<int64_t>(npix, 1) * 4, st));
  int32_t* last = static_cast<int32_t*>(ctx->last.get((size_t)std::max<int64_t>(npix, 1) * 4, st));
  if (o.meta) {
    o.meta[0] = w.px0; o.meta[1] = w.py0; o.meta[2] = w.pw; o.meta[3] = w.ph; o.meta[4] = V; o.meta[5] = ctx->I;
  }
  if (npix == 0) {
    if (o.gt) GSS_CUDA(cudaMemsetAsync(o.loss_dev, 0, sizeof(float), st));
    if (o.gt && o.loss_sum) GSS_CUDA(cudaMemsetAsync(o.loss_sum, 0, sizeof(double), st));
    return;
  }
  const int ntile = w.tw * w.th;
  double* lp = o.gt ? static_cast<double*>(ctx->lossp.get((size_t)ntile * 8, st)) : nullptr;
  ktime_begin(ctx, 0, st);
  forward_kernel<<<ntile, kFwdThreads, 0, st>>>(static_cast<const SplatRec*>(ctx->recs.p),
                                             static_cast<const int32_t*>(ctx->vals_a.p),
                                             static_cast<const int2*>(ctx->ranges.p),
                                             static_cast<const int32_t*>(ctx->tile_order.p), w, s.bg[0], s.bg[1], s.bg[2],
                                             o.image, fT, last, o.ncontrib, o.gt, o.gt_width, o.inv, o.d_img, lp,
                                             ctx->ktiming ? ctx->contribs_dev : nullptr, exp_coef_host());
  GSS_LAUNCHED();
  ktime_end(ctx, st);
  if (o.gt) {
    loss_final_kernel<<<1, 1024, 0, st>>>(lp, ntile, o.inv, o.loss_dev, o.loss_sum);
    GSS_LAUNCHED();
  }
  if (o.final_T) GSS_CUDA(cudaMemcpyAsync(o.final_T, fT, npix * 4, cudaMemcpyDeviceToDevice, st));
}

void bin_and_composite(gss_render_ctx* ctx, const Win& w, int64_t V, const FwdOut& o, cudaStream_t st) {
  bin_phase(ctx, w, V, st);
  composite_phase(ctx, w, V, o, st);
}

void begin_forward(gss_render_ctx* ctx, const gss_camera* cam, const Win& w, int64_t V, cudaStream_t st) {
  ctx->last_stream = st;
  std::memcpy(&ctx->cam, cam, sizeof(Cam));
  ctx->win = w;
  ctx->V = V;
  ctx->I = 0;
  ctx->pay_sorted = nullptr;
  ctx->have_forward = 1;
}

void alloc_records(gss_render_ctx* ctx, int64_t V, cudaStream_t st) {
  const size_t n = (size_t)std::max<int64_t>(V, 1);
  ctx->recs.get(n * sizeof(SplatRec), st);
  ctx->ntiles.get((n + 1) * 4, st);
  ctx->dkeys_a.get(n * 4, st);
  ctx->order_a.get(n * 8, st);  // depth-sort payloads (slot + packed tile box)
}

void per_slot_sums(gss_render_ctx* ctx, const float* d_img, float* sums, cudaStream_t st) {
  const Win& w = ctx->win;
  const int64_t V = ctx->V, I = ctx->I;
  const int64_t npix = (int64_t)w.pw * w.ph;
  require(npix == 0 || d_img, "rasterize_backward: null d_img");
  if (I == 0 || npix == 0) {  // no tile instances: every per-slot sum is zero
    GSS_CUDA(cudaMemsetAsync(sums, 0, (size_t)V * 9 * 4, st));
    return;
  }
  const SplatRec* recs = static_cast<const SplatRec*>(ctx->recs.p);
  const int32_t* soff = static_cast<const int32_t*>(ctx->slot_off.p);
  const int32_t* nts = static_cast<const int32_t*>(ctx->ntiles.p);
  // every instance partial is written by the sweep (walked records, or zeros for a tile's T-stop tail)
  float* partials = static_cast<float*>(ctx->partials.get((size_t)std::max<int64_t>(I, 1) * 9 * 4, st));
  {
    const int ntile = w.tw * w.th;
    ktime_begin(ctx, 1, st);
    backward_kernel<<<ntile, kBwdThreads, 0, st>>>(recs, static_cast<const int32_t*>(ctx->vals_a.p),
                                                static_cast<const int2*>(ctx->ranges.p),
                                                static_cast<const int32_t*>(ctx->tile_order.p), w, ctx->sc.bg[0],
                                                ctx->sc.bg[1], ctx->sc.bg[2], static_cast<const float*>(ctx->fT.p),
                                                static_cast<const int32_t*>(ctx->last.p), d_img, partials);
    GSS_LAUNCHED();
    ktime_end(ctx, st);
  }
#ifndef GSS_SUM_DEPTH
#define GSS_SUM_DEPTH 1
#endif
  ktime_begin(ctx, 4, st);
  if (GSS_SUM_DEPTH && ctx->pay_sorted) {
    // slots never binned (V_bin .. V in depth order: depth key 0xffffffff) have no instances: their
    // ranges are empty and their sums are written as zeros like every other slot's
    if (GSS_SUM_SEG)
      slot_sum_seg_kernel<<<(unsigned)ceil_div(V, kSumWarps * 32), kSumWarps * 32, 0, st>>>(
          V, static_cast<const int32_t*>(ctx->offsets.p), ctx->pay_sorted, partials, sums);
    else
      slot_sum_depth_kernel<<<(unsigned)ceil_div(V, kSumWarps * 32), kSumWarps * 32, 0, st>>>(
          V, static_cast<const int32_t*>(ctx->offsets.p), ctx->pay_sorted, partials, sums);
  } else {
    slot_sum_kernel<<<(unsigned)ceil_div(V, kSumThreads), kSumThreads, 0, st>>>(V, soff, nts, partials, sums);
  }
  GSS_LAUNCHED();
  ktime_end(ctx, st);
}

void launch_chain(const SceneDev& sc, const Cam& cam, const Win& w, int64_t V, const SplatRec* recs, const float* sums,
                  float* gg, int64_t gstride, float* gn, int64_t nstride, float* mean2d, cudaStream_t st) {
  const unsigned cb = (unsigned)ceil_div(V, kChainThreads);
  switch (sc.sh_degree) {
    case 0: chain_kernel<0><<<cb, kChainThreads, 0, st>>>(sc, cam, w, V, recs, sums, gg, gstride, gn, nstride, mean2d); break;
    case 1: chain_kernel<1><<<cb, kChainThreads, 0, st>>>(sc, cam, w, V, recs, sums, gg, gstride, gn, nstride, mean2d); break;
    case 2: chain_kernel<2><<<cb, kChainThreads, 0, st>>>(sc, cam, w, V, recs, sums, gg, gstride, gn, nstride, mean2d); break;
    default: chain_kernel<3><<<cb, kChainThreads, 0, st>>>(sc, cam, w, V, recs, sums, gg, gstride, gn, nstride, mean2d); break;
  }
  GSS_LAUNCHED();
}

}  // namespace

void rasterize_forward(gss_render_ctx* ctx, const gss_render_scene* scene, const gss_camera* cam,
                       const gss_viewport* vp, float* image, const float* gt, int64_t normalizer, float* d_img,
                       float* loss_dev, float* final_T_opt, int32_t* ncontrib_opt, int64_t* meta, cudaStream_t st) {
  require(ctx && scene && cam && vp && image, "rasterize_forward: null argument");
  require(!gt || (d_img && loss_dev), "rasterize_forward: gt needs d_img and loss_dev");
  set_scene(ctx, scene);
  if (!ctx->pinned) GSS_CUDA(cudaMallocHost(&ctx->pinned, 4 * sizeof(int64_t)));
  const Win w = make_window(*vp);
  require(!gt || (w.px0 + w.pw <= cam->width && w.py0 + w.ph <= cam->height),
          "compute_loss_l1: image and ground-truth shapes differ");
  const int64_t V = scene_count(ctx, scene, st);
  begin_forward(ctx, cam, w, V, st);
  const int64_t npix = (int64_t)w.pw * w.ph;
  const float inv = gt ? 1.0f / (float)(double)(normalizer > 0 ? normalizer : npix * 3) : 0.0f;
  alloc_records(ctx, V, st);
  if (V > 0 && npix > 0) {
    preprocess_kernel<true><<<(unsigned)ceil_div(V, 128), 128, 0, st>>>(
        ctx->sc, ctx->cam, w, V, static_cast<SplatRec*>(ctx->recs.p), static_cast<int32_t*>(ctx->ntiles.p),
        static_cast<uint32_t*>(ctx->dkeys_a.p), static_cast<uint64_t*>(ctx->order_a.p));
    GSS_LAUNCHED();
  }
  bin_and_composite(ctx, w, V, FwdOut{image, gt, cam->width, inv, d_img, loss_dev, nullptr, final_T_opt, ncontrib_opt,
                                      meta}, st);
}

void loss_l1(const float* image, const float* gt, int64_t elems, int64_t normalizer, float* d_img, float* loss_dev,
             cudaStream_t st) {
  require(elems >= 0 && (elems == 0 || (image && gt && d_img)) && loss_dev, "compute_loss_l1: null argument");
  if (normalizer == 0) normalizer = elems;
  const float inv = 1.0f / (float)(double)normalizer;
  if (elems == 0) {
    GSS_CUDA(cudaMemsetAsync(loss_dev, 0, sizeof(float), st));
    return;
  }
  const int blocks = (int)std::min<int64_t>(ceil_div(elems, 256), 1024);
  double* lp = nullptr;
  GSS_CUDA(cudaMallocAsync((void**)&lp, (size_t)blocks * 8, st));
  loss_partial_kernel<<<blocks, 256, 0, st>>>(image, gt, elems, inv, d_img, lp);
  GSS_LAUNCHED();
  loss_final_kernel<<<1, 1024, 0, st>>>(lp, blocks, inv, loss_dev, nullptr);
  GSS_LAUNCHED();
  GSS_CUDA(cudaFreeAsync(lp, st));
}

void image_sq_err(const float* a, const float* b, int64_t elems, double* sum_dev, cudaStream_t st) {
  require(elems >= 0 && sum_dev && (elems == 0 || (a && b)), "image_sq_err: null argument");
  if (elems == 0) {
    GSS_CUDA(cudaMemsetAsync(sum_dev, 0, sizeof(double), st));
    return;
  }
  const int blocks = (int)std::min<int64_t>(ceil_div(elems, 256), 1024);
  double* lp = nullptr;
  GSS_CUDA(cudaMallocAsync((void**)&lp, (size_t)blocks * 8, st));
  sq_err_partial_kernel<<<blocks, 256, 0, st>>>(a, b, elems, lp);
  GSS_LAUNCHED();
  sum_partials_kernel<<<1, 1024, 0, st>>>(lp, blocks, sum_dev);
  GSS_LAUNCHED();
  GSS_CUDA(cudaFreeAsync(lp, st));
}

void rasterize_backward(gss_render_ctx* ctx, const float* d_img, float* gg, int64_t gstride, float* gn,
                        int64_t nstride, float* mean2d, cudaStream_t st) {
  require(ctx && ctx->have_forward, "rasterize_backward: no forward result in this context");
  require(gstride >= 10 && nstride >= 49, "rasterize_backward: bad gradient strides");
  const int64_t V = ctx->V;
  if (V == 0) return;
  require(gg && gn, "rasterize_backward: null gradient buffers");
  float* sums = static_cast<float*>(ctx->sums.get((size_t)V * 9 * 4, st));
  per_slot_sums(ctx, d_img, sums, st);
  ktime_begin(ctx, 5, st);
  launch_chain(ctx->sc, ctx->cam, ctx->win, V, static_cast<const SplatRec*>(ctx->recs.p), sums, gg, gstride, gn,
               nstride, mean2d, st);
  ktime_end(ctx, st);
}

// Two-phase forward for the engine: the geometry half (projection, depth/tile sort, tile ranges)
// needs only the geometric tier, so it runs while the forwarding gather of the non-geometric rows
// is still in flight on the other stream; finish() adds opacity/colour and composites.
void rasterize_forward_geometry(gss_render_ctx* ctx, const gss_render_scene* scene, const gss_camera* cam,
                                const gss_viewport* vp, cudaStream_t st) {
  require(ctx && scene && cam && vp, "rasterize_forward: null argument");
  ktime_begin(ctx, 2, st);
  set_scene(ctx, scene);
  if (!ctx->pinned) GSS_CUDA(cudaMallocHost(&ctx->pinned, 4 * sizeof(int64_t)));
  const Win w = make_window(*vp);
  const int64_t V = scene_count(ctx, scene, st);
  begin_forward(ctx, cam, w, V, st);
  alloc_records(ctx, V, st);
  if (V > 0 && (int64_t)w.pw * w.ph > 0) {
    preprocess_kernel<false><<<(unsigned)ceil_div(V, 128), 128, 0, st>>>(
        ctx->sc, ctx->cam, w, V, static_cast<SplatRec*>(ctx->recs.p), static_cast<int32_t*>(ctx->ntiles.p),
        static_cast<uint32_t*>(ctx->dkeys_a.p), static_cast<uint64_t*>(ctx->order_a.p));
    GSS_LAUNCHED();
  }
  bin_phase(ctx, w, V, st);
  ktime_end(ctx, st);
}

void rasterize_forward_finish(gss_render_ctx* ctx, float* image, const float* gt, int64_t normalizer, float* d_img,
                              float* loss_dev, cudaStream_t st) {
  require(ctx && ctx->have_forward && image, "rasterize_forward: no geometry phase / null image");
  require(!gt || (d_img && loss_dev), "rasterize_forward: gt needs d_img and loss_dev");
  const Win& w = ctx->win;
  const int64_t V = ctx->V;
  const int64_t npix = (int64_t)w.pw * w.ph;
  require(!gt || (w.px0 + w.pw <= ctx->cam.width && w.py0 + w.ph <= ctx->cam.height),
          "compute_loss_l1: image and ground-truth shapes differ");
  const float inv = gt ? 1.0f / (float)(double)(normalizer > 0 ? normalizer : npix * 3) : 0.0f;
  if (V > 0 && npix > 0) {
    ktime_begin(ctx, 3, st);
    auto ck = ctx->sc.sh_degree == 0 ? colour_kernel<0>
              : ctx->sc.sh_degree == 1 ? colour_kernel<1>
              : ctx->sc.sh_degree == 2 ? colour_kernel<2> : colour_kernel<3>;
    ck<<<(unsigned)ceil_div(V, kColThreads), kColThreads, 0, st>>>(ctx->sc, ctx->cam, V,
                                                              static_cast<const int32_t*>(ctx->ntiles.p),
                                                              static_cast<SplatRec*>(ctx->recs.p));
    GSS_LAUNCHED();
    ktime_end(ctx, st);
  }
  composite_phase(ctx, w, V, FwdOut{image, gt, ctx->cam.width, inv, d_img, loss_dev, nullptr, nullptr, nullptr,
                                    nullptr}, st);
}

// ---- split-phase rasterizer for image-parallel rendering ----------------------

void project(const gss_render_scene* scene, const gss_camera* cam, const gss_viewport* vp, void* records,
             cudaStream_t st) {
  require(scene && cam && vp && (scene->count == 0 || records), "project: null argument");
  require(!scene->count_dev, "project: needs a host-known count");
  gss_render_ctx tmp;
  set_scene(&tmp, scene);
  const int64_t V = scene->count;
  require(V >= 0 && V <= INT32_MAX, "project: visible count out of range");
  if (V == 0) return;
  Cam c;
  std::memcpy(&c, cam, sizeof(Cam));
  preprocess_kernel<true><<<(unsigned)ceil_div(V, 128), 128, 0, st>>>(tmp.sc, c, make_window(*vp), V,
                                                                static_cast<SplatRec*>(records), nullptr, nullptr,
                                                                nullptr);
  GSS_LAUNCHED();
}

void route_strips(const void* records, int64_t count, const int32_t* strip_x, int nstrips, int32_t* dest_slots,
                  int64_t* dest_counts, cudaStream_t st) {
  require(count >= 0 && count <= INT32_MAX && nstrips >= 1, "route_strips: bad sizes");
  require(strip_x && dest_counts && (count == 0 || (records && dest_slots)), "route_strips: null argument");
  for (int k = 0; k < nstrips; ++k) require(strip_x[k] <= strip_x[k + 1], "route_strips: strips must ascend");
  if (count == 0) {
    GSS_CUDA(cudaMemsetAsync(dest_counts, 0, (size_t)nstrips * 8, st));
    return;
  }
  const SplatRec* recs = static_cast<const SplatRec*>(records);
  size_t tb = 0;
  thrust::counting_iterator<int32_t> it(0);
  GSS_CUDA(cub::DeviceSelect::If(nullptr, tb, it, dest_slots, dest_counts, (int)count,
                                 StripHit{recs, strip_x[0], strip_x[1]}, st));
  void* tmp = nullptr;
  GSS_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tb, 16), st));
  for (int k = 0; k < nstrips; ++k) {
    GSS_CUDA(cub::DeviceSelect::If(tmp, tb, it, dest_slots + (size_t)k * count, dest_counts + k, (int)count,
                                   StripHit{recs, strip_x[k], strip_x[k + 1]}, st));
    count_launch();
  }
  GSS_CUDA(cudaFreeAsync(tmp, st));
}

void gather_records(const void* records, const int32_t* slots, int64_t n, void* out, cudaStream_t st) {
  require(n >= 0 && (n == 0 || (records && slots && out)), "gather_records: null argument");
  if (n == 0) return;
  gather_records_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(static_cast<const SplatRec*>(records), slots, n,
                                                                    static_cast<SplatRec*>(out));
  GSS_LAUNCHED();
}

void scatter_add_rows(const float* src, const int32_t* slots, int64_t n, int width, float* dst, cudaStream_t st) {
  require(n >= 0 && width > 0 && (n == 0 || (src && slots && dst)), "scatter_add_rows: null argument");
  if (n == 0) return;
  scatter_add_rows_kernel<<<(unsigned)ceil_div(n * width, 256), 256, 0, st>>>(src, slots, n, width, dst);
  GSS_LAUNCHED();
}

void rasterize_records_forward(gss_render_ctx* ctx, const void* records, int64_t count, const gss_camera* cam,
                               const gss_viewport* vp, const float* background, float* image, const float* gt,
                               int64_t normalizer, float* d_img, float* loss_dev, double* loss_sum_dev,
                               float* final_T_opt, int32_t* ncontrib_opt, int64_t* meta, cudaStream_t st) {
  require(ctx && cam && vp && background && (count == 0 || records), "rasterize_records_forward: null argument");
  require(count >= 0 && count <= INT32_MAX, "rasterize_records_forward: count out of range");
  if (!ctx->pinned) GSS_CUDA(cudaMallocHost(&ctx->pinned, 4 * sizeof(int64_t)));
  const Win w = make_window(*vp);
  const bool empty = (int64_t)w.pw * w.ph == 0;  // an empty strip: no pixel buffers needed
  require(empty || image, "rasterize_records_forward: null image");
  require(!gt || ((empty || d_img) && loss_dev), "rasterize_records_forward: gt needs d_img and loss_dev");
  require(!gt || (w.px0 + w.pw <= cam->width && w.py0 + w.ph <= cam->height),
          "compute_loss_l1: image and ground-truth shapes differ");
  ctx->sc = SceneDev{};
  for (int c = 0; c < 3; ++c) ctx->sc.bg[c] = background[c];
  begin_forward(ctx, cam, w, count, st);
  const int64_t npix = (int64_t)w.pw * w.ph;
  const float inv = gt ? 1.0f / (float)(double)(normalizer > 0 ? normalizer : npix * 3) : 0.0f;
  alloc_records(ctx, count, st);
  if (count > 0 && npix > 0) {
    clip_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(
        static_cast<const SplatRec*>(records), count, w, static_cast<SplatRec*>(ctx->recs.p),
        static_cast<int32_t*>(ctx->ntiles.p), static_cast<uint32_t*>(ctx->dkeys_a.p),
        static_cast<uint64_t*>(ctx->order_a.p));
    GSS_LAUNCHED();
  }
  bin_and_composite(ctx, w, count, FwdOut{image, gt, cam->width, inv, d_img, loss_dev, loss_sum_dev, final_T_opt,
                                          ncontrib_opt, meta}, st);
}

void rasterize_records_backward(gss_render_ctx* ctx, const float* d_img, float* sums, cudaStream_t st) {
  require(ctx && ctx->have_forward, "rasterize_records_backward: no forward result in this context");
  if (ctx->V == 0) return;
  require(sums, "rasterize_records_backward: null sums");
  per_slot_sums(ctx, d_img, sums, st);
}

void chain_backward(const gss_render_scene* scene, const gss_camera* cam, const void* records, const float* sums,
                    float* gg, int64_t gstride, float* gn, int64_t nstride, float* mean2d, cudaStream_t st) {
  require(scene && cam && (scene->count == 0 || (records && sums && gg && gn)), "chain_backward: null argument");
  require(!scene->count_dev, "chain_backward: needs a host-known count");
  require(gstride >= 10 && nstride >= 49, "chain_backward: bad gradient strides");
  gss_render_ctx tmp;
  set_scene(&tmp, scene);
  if (scene->count == 0) return;
  Cam c;
  std::memcpy(&c, cam, sizeof(Cam));
  launch_chain(tmp.sc, c, Win{}, scene->count, static_cast<const SplatRec*>(records), sums, gg, gstride, gn, nstride,
               mean2d, st);
}

gss_render_ctx* render_ctx_create() { return new gss_render_ctx(); }

void render_ctx_destroy(gss_render_ctx* ctx) {
  if (!ctx) return;
  cudaStream_t st = ctx->last_stream;
  for (DBuf* b : {&ctx->recs, &ctx->ntiles, &ctx->offsets, &ctx->keys_a, &ctx->keys_b, &ctx->vals_a, &ctx->vals_b,
                  &ctx->cub_tmp, &ctx->ranges, &ctx->tile_order, &ctx->last, &ctx->fT, &ctx->partials, &ctx->lossp, &ctx->hostcnt, &ctx->sums, &ctx->dkeys_a, &ctx->dkeys_b, &ctx->order_a, &ctx->order_b,
                  &ctx->slot_off})
    b->release(st);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  cudaDeviceSynchronize();
  for (auto& t : ctx->ktimes) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : ctx->kfree) cudaEventDestroy(e);
  if (ctx->contribs_dev) cudaFree(ctx->contribs_dev);
  cudaGetLastError();
  delete ctx;
}

// Live per-kernel timing of the composite (forward_kernel) and sweep (backward_kernel) launches.
void render_ctx_timing(gss_render_ctx* ctx, bool on) {
  require(ctx != nullptr, "render ctx: null");
  ctx->ktiming = on;
  if (on && !ctx->contribs_dev) {
    GSS_CUDA(cudaMalloc(&ctx->contribs_dev, sizeof(unsigned long long)));
    GSS_CUDA(cudaMemset(ctx->contribs_dev, 0, sizeof(unsigned long long)));
  }
}
// Folds the recorded intervals (all must have completed: call after a sync) into
// out[0..1] = total ms of forward_kernel / backward_kernel launches, n[0..1] = launches,
// *contribs = composited contributions; resets the accumulators.
void render_ctx_times(gss_render_ctx* ctx, double* ms2, int64_t* n2, uint64_t* contribs, int nk) {
  require(ctx != nullptr, "render ctx: null");
  for (auto& t : ctx->ktimes) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
      ctx->kms[t.kind] += ms;
      ctx->kn[t.kind] += 1;
    }
    ctx->kfree.push_back(t.a);
    ctx->kfree.push_back(t.b);
  }
  cudaGetLastError();
  ctx->ktimes.clear();
  for (int k = 0; k < gss_render_ctx::kKinds; ++k) {
    if (ms2 && k < nk) ms2[k] = ctx->kms[k];
    if (n2 && k < nk) n2[k] = ctx->kn[k];
    ctx->kms[k] = 0.0;
    ctx->kn[k] = 0;
  }
  unsigned long long c = 0;
  if (ctx->contribs_dev) {
    GSS_CUDA(cudaMemcpy(&c, ctx->contribs_dev, sizeof c, cudaMemcpyDeviceToHost));
    GSS_CUDA(cudaMemset(ctx->contribs_dev, 0, sizeof c));
  }
  if (contribs) *contribs = c;
}

// Work-accounting counters of the rasterizer kernels (see g_rstats); all zero unless the library was
// built with GSS_RASTER_STATS=1.
void raster_stats(uint64_t* out8, bool reset) {
  unsigned long long h[8];
  GSS_CUDA(cudaMemcpyFromSymbol(h, g_rstats, sizeof h));
  for (int i = 0; i < 8; ++i) out8[i] = h[i];
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    GSS_CUDA(cudaMemcpyToSymbol(g_rstats, z, sizeof z));
  }
}
int raster_stats_enabled() { return GSS_RASTER_STATS; }

}  // namespace gssd
