// OffloadEngine on the B200 (reference: engine.hpp:55-522, store.hpp:149-248).
//
// The reference runs six stages on two std::threads (a "device" worker and a "host" worker)
// synchronised by condition-variable Events; here the two workers are two CUDA streams and the
// Events are cudaEvents, enqueued by one host thread:
//   stream D: cull(g) -> render(g) -> geo_update(g) -> handoff(g)
//   stream H: forward_params(g) -> lazy_update(g-1)
// with the reference's edges (engine.hpp:477-516): fp(g) waits cull(g) and handoff(g-1);
// render(g) waits fp(g); lazy(g-1) runs after fp(g) on H, overlapping render(g) on D.
// Serial mode issues the same stages on one stream in run_serial's order. Every kernel is
// deterministic, so serial and pipelined trajectories are bitwise identical.
//
// Tier placement (selective offloading, store.hpp:149-192): the geometric tier (N x 10 w/m/v,
// geo_defer_max = 0 => dense immediate update) lives in HBM. The non-geometric tier (N x 49
// w/m/v + uint8 counters, defer_max) lives in HBM (scene fits: 180 GB) or, with
// nongeo_on_host, in pinned host memory read by the forwarding gather through the PCIe/C2C
// mapping and updated lazily in place (zero-copy), see DESIGN.md §offload.
#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "common.cuh"
#include "gss_math.cuh"

namespace gssd {
void cull(const float* geo, int64_t n, int64_t stride, const gss_camera* cam, const gss_viewport* vp, float lp,
          uint32_t* mask, int32_t* ids, int64_t* count, void* ws, size_t ws_bytes, cudaStream_t st);
size_t cull_workspace_bytes(int64_t n);
void adam_update(gss_arena* ap, const gss_sparse_grads* grads, int32_t* touched_ids, int64_t* touched_count,
                 cudaStream_t st, const uint32_t* split_mask = nullptr, cudaEvent_t split_before_set = nullptr);
void adam_restore(const gss_arena* ap, const int32_t* ids, int64_t count, const int64_t* count_dev,
                  const gss_sparse_grads* pending, float* out, cudaStream_t st, cudaEvent_t after_resolve = nullptr);
void rasterize_forward(gss_render_ctx* ctx, const gss_render_scene* scene, const gss_camera* cam,
                       const gss_viewport* vp, float* image, const float* gt, int64_t normalizer, float* d_img,
                       float* loss_dev, float* final_T_opt, int32_t* ncontrib_opt, int64_t* meta, cudaStream_t st);
void plan_densify(const float* rows, int64_t n, const double* norm, const int32_t* cnt,
                  const gss_densify_config* dc, double extent, uint64_t seed, int32_t* survivors, float* children,
                  int64_t* counts, cudaStream_t st);
void rasterize_forward_geometry(gss_render_ctx* ctx, const gss_render_scene* scene, const gss_camera* cam,
                                const gss_viewport* vp, cudaStream_t st);
void rasterize_forward_finish(gss_render_ctx* ctx, float* image, const float* gt, int64_t normalizer, float* d_img,
                              float* loss_dev, cudaStream_t st);
void rasterize_backward(gss_render_ctx* ctx, const float* d_img, float* gg, int64_t gstride, float* gn,
                        int64_t nstride, float* mean2d, cudaStream_t st);
void render_ctx_destroy(gss_render_ctx* ctx);
gss_render_ctx* render_ctx_create();
void arena_release(const gss_arena* ap);
void render_ctx_timing(gss_render_ctx* ctx, bool on);
void render_ctx_times(gss_render_ctx* ctx, double* ms2, int64_t* n2, uint64_t* contribs, int nk);
void set_host_chunk_bytes(int64_t bytes);
}  // namespace gssd

struct gss_render_ctx;

namespace gssd {
namespace {

constexpr int kGeoDim = 10, kNgDim = 49, kRowDim = 59;
// Non-geometric tier layout: w, m, v of a row interleaved in one 640-byte span (5 x 128-byte
// lines: w at 0, m at 52, v at 104, each segment 16-byte aligned and padded to 13 float4), so a
// touched row of the deferred update / forwarding gather is five whole cache lines walked with
// 16-byte accesses instead of three scattered 196-byte rows.
constexpr int kNgStride = 160, kNgSeg = 52;
// Gradient stage rows of the non-geometric tier: 52 floats (16-byte aligned, the deferred pass's TMA
// gathers them whole).
constexpr int kNgGradStride = 52;

__global__ void handoff_stats_kernel(const int32_t* ids, const int64_t* count, const float* mean2d, double* norm,
                                     int32_t* cnt) {
  const int64_t V = *count;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < V; k += (int64_t)gridDim.x * blockDim.x) {
    const double gx = (double)mean2d[k * 2], gy = (double)mean2d[k * 2 + 1];
    const int id = ids[k];
    norm[id] += sqrt(gx * gx + gy * gy);  // engine.hpp:404-408
    cnt[id] += 1;
  }
}

__global__ void split_rows_kernel(const float* rows, int64_t n, float* geo, float* ng) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * kRowDim) return;
  const int64_t r = i / kRowDim;
  const int c = (int)(i - r * kRowDim);
  if (c < kGeoDim) geo[r * kGeoDim + c] = rows[i]; else ng[r * kNgStride + (c - kGeoDim)] = rows[i];
}

__global__ void join_rows_kernel(const float* geo, const float* ng, int64_t n, float* rows) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * kRowDim) return;
  const int64_t r = i / kRowDim;
  const int c = (int)(i - r * kRowDim);
  rows[i] = c < kGeoDim ? geo[r * kGeoDim + c] : ng[r * kNgDim + (c - kGeoDim)];
}

__global__ void iota_kernel(int32_t* ids, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) ids[i] = (int32_t)i;
}

// Sets (on) or clears the row bits of a sorted id list in a row bit mask.
__global__ void mark_rows_kernel(const int32_t* ids, const int64_t* count, uint32_t* mask, int on) {
  const int64_t V = *count;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < V; k += (int64_t)gridDim.x * blockDim.x) {
    const int id = ids[k];
    if (on) atomicOr(&mask[id >> 5], 1u << (id & 31));
    else atomicAnd(&mask[id >> 5], ~(1u << (id & 31)));
  }
}

// ---- split cameras: std::set_union of the two sorted cull lists (engine.hpp:270-272) and the
// slot maps of each side into the union (engine.hpp:324-332), from the two cull bit masks.
// popc(left | right) per 32-row word; word nwords holds 0 so the scan's last entry is the count.
__global__ void union_popc_kernel(const uint32_t* L, const uint32_t* R, int64_t nwords, int32_t* wc) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w < nwords) wc[w] = __popc(L[w] | R[w]);
  else if (w == nwords) wc[w] = 0;
}
// Union ids ascending: word w's set bits at wpre[w] + rank within the word; count = wpre[nwords].
__global__ void union_ids_kernel(const uint32_t* L, const uint32_t* R, const int32_t* wpre, int64_t nwords,
                                 int32_t* ids, int64_t* count) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w == nwords) *count = wpre[nwords];
  if (w >= nwords) return;
  uint32_t u = L[w] | R[w];
  int32_t o = wpre[w];
  while (u) {
    const int b = __ffs(u) - 1;
    u &= u - 1;
    ids[o++] = (int32_t)(w * 32 + b);
  }
}
// slot of sub-list entry k in the union = number of union ids below it.
__global__ void union_slot_kernel(const int32_t* sub, const int64_t* sub_count, const uint32_t* L, const uint32_t* R,
                                  const int32_t* wpre, int32_t* map) {
  const int64_t V = *sub_count;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < V; k += (int64_t)gridDim.x * blockDim.x) {
    const int id = sub[k];
    const int w = id >> 5;
    const uint32_t below = (L[w] | R[w]) & ((1u << (id & 31)) - 1u);
    map[k] = wpre[w] + __popc(below);
  }
}
// aggregate_grads (splitter.hpp:85-123): out[map[k]] += in[k] over `width` columns; the left side
// is added before the right (two launches in order) onto zeroed rows, the reference's
// `row = 0; row += left; row += right` arithmetic.
__global__ void add_rows_kernel(const float* in, int64_t stride, const int32_t* map, const int64_t* count, int width,
                                float* out) {
  const int64_t n = *count * width;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / width;
    const int c = (int)(e - k * width);
    out[(int64_t)map[k] * stride + c] += in[k * stride + c];
  }
}
// loss = ll + rl (engine.hpp:362).
__global__ void split_loss_kernel(const float* sl, float* loss) { *loss = sl[0] + sl[1]; }

template <class T> T* dmalloc(size_t count) {
  T* p = nullptr;
  if (count == 0) count = 1;
  GSS_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

struct Ev {
  cudaEvent_t e = nullptr;
  Ev() { GSS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~Ev() { if (e) cudaEventDestroy(e); }
};

enum Stage { kCull = 0, kFwd, kRender, kGeo, kHandoff, kLazy, kStages };
const char* const kStageName[kStages] = {"cull", "forward_params", "render", "geo_update", "handoff", "lazy_update"};

// Test instrumentation (the reference's EngineConfig::stage_hook delays, engine.hpp:42-43,
// test_offload.cpp:268-285): a device-side sleep at the start of a stage on the stage's stream.
__global__ void stage_delay_kernel(uint32_t ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
    __nanosleep(1000);
  }
}

}  // namespace
}  // namespace gssd

struct gss_engine {
  gss_engine_config cfg{};
  int64_t n = 0;
  std::vector<gss_camera> cams;
  float* gts_dev = nullptr;  // ncams x H x W x 3 (optional)
  int W = 0, H = 0;
  // tiers
  float *gw = nullptr, *gm = nullptr, *gv = nullptr;
  uint8_t* gcnt = nullptr;
  float *nw = nullptr, *nm = nullptr, *nv = nullptr;
  uint8_t* ncnt = nullptr;
  bool ng_host = false;
  gss_arena geo{}, ng{};
  // plans: ring of 3 (engine.hpp:195-203)
  int32_t* ids[3] = {nullptr, nullptr, nullptr};
  int64_t* count[3] = {nullptr, nullptr, nullptr};
  int64_t* count_host = nullptr;  // pinned [3]
  void* cull_ws = nullptr;
  size_t cull_ws_bytes = 0;
  // forward stage (double-buffered, engine.hpp:211)
  float* fwd[2] = {nullptr, nullptr};
  int fwd_iter[2] = {-1, -1};
  // gradient stage (double-buffered GradStage, store.hpp:227-248)
  float* g_geo[2] = {nullptr, nullptr};
  float* g_ng[2] = {nullptr, nullptr};
  float* g_m2d[2] = {nullptr, nullptr};
  int g_iter[2] = {-1, -1};
  int g_plan[2] = {-1, -1};
  int64_t cap_rows = 0;  // capacity of fwd / grad buffers in rows
  // render
  gss_render_ctx* rctx = nullptr;
  float* image = nullptr;
  float* d_img = nullptr;
  float* gt_step[2] = {nullptr, nullptr};  // step(): double-buffered ground truth
  int gt_cur = 0;
  float* loss_dev = nullptr;  // per iteration of a run
  int loss_cap = 0;
  double* accum_norm = nullptr;
  int32_t* accum_cnt = nullptr;
  // streams / events
  cudaStream_t sD = nullptr, sH = nullptr, sC = nullptr;  // sC: host->device ground-truth copies of step()
  gssd::Ev ev_cull[3], ev_fp[2], ev_handoff[2], ev_lazy[2], ev_render[2], ev_gt, ev_gt_done[2];
  // host tier, concurrent forwarding: the lazy update runs on its own stream sL beside the
  // forwarding gather of the next iteration (disjoint rows; see stage_lazy)
  cudaStream_t sL = nullptr;
  gssd::Ev ev_resolved[2];        // fp(g)'s resolve pass (counters read) done
  uint32_t* vis_mask = nullptr;   // bit per row: in the visible set of the iteration being forwarded
  bool gt_pending = false;  // render must wait for ev_gt (the step's ground truth in flight)
  struct TimeRec {
    int stage;
    cudaEvent_t a, b;
    int iter;
    int worker;      // 0: device stream (stream D), 1: host-tier stream (stream H), as TimelineRow::worker
    uint64_t bytes;  // algorithmic bytes of the stage (lazy update from its touched count)
    int touched_slot;
  };
  std::vector<cudaEvent_t> ev_free;
  std::vector<TimeRec> pending_times;
  double stage_ms[gssd::kStages] = {0, 0, 0, 0, 0, 0};
  // Per-iteration timeline (engine.hpp:22-28, 230-237): rows are kept when enabled; times are
  // CUDA-event offsets from the epoch event recorded when the timeline was enabled.
  bool timeline_on = false;
  cudaEvent_t epoch = nullptr;
  std::vector<gss_timeline_row> timeline;
  int64_t* touched_ring = nullptr;  // device: touched counts of the lazy updates in flight
  int touched_next = 0;
  std::vector<uint32_t> delays_ns;  // stage-delay injection (test instrumentation)
  size_t delay_next = 0;
  // iteration bookkeeping
  // split cameras (engine.hpp:62-68, 266-273, 356-371): per stored camera the split column
  // (-1 = rendered whole). Left / right culls, their union and the slot maps live per plan.
  std::vector<int32_t> split_col;
  int plan_col[3] = {-1, -1, -1};
  int64_t split_cap = 0;                 // capacity (rows) of the split buffers
  uint32_t* smask[2] = {nullptr, nullptr};  // left / right cull masks (stream D scratch)
  int32_t* wpre = nullptr;               // exclusive prefix of popc(left | right) per mask word
  void* scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;
  int32_t* sids[3][2] = {};              // per plan: left / right ids
  int32_t* smap[3][2] = {};              // per plan: left / right slot -> union slot
  int64_t* scount[3][2] = {};            // per plan: left / right counts (device)
  int64_t* scount_host = nullptr;        // pinned [3][2]
  int64_t scap_rows = 0;                 // capacity of the per-side gradient buffers
  float* sg_geo[2] = {nullptr, nullptr};
  float* sg_ng[2] = {nullptr, nullptr};
  float* sg_m2d[2] = {nullptr, nullptr};
  float* sloss = nullptr;                // [2] per-side losses of the iteration being rendered
  int next_iter = 0;
  int seg_begin = 0;
  int open_pending = -1;  // iteration whose lazy update is still owed
  int64_t launches_at_start = 0, launches_last = 0;
  std::vector<int64_t> valid_counts;
};

namespace gssd {
namespace {

cudaStream_t S(gss_engine* e, bool host_tier) { return (e->cfg.pipelined && host_tier) ? e->sH : e->sD; }

// The pinned host tier with the lazy update of g-1 beside the forwarding gather of g (both
// link-bound; GSS_HOST_CONCURRENT=0 keeps them in the reference's serial order on stream H).
bool host_concurrent(const gss_engine* e) {
  static const bool on = [] {
    const char* v = std::getenv("GSS_HOST_CONCURRENT");
    return !(v && v[0] == '0');
  }();
  return e->ng_host && e->cfg.pipelined && e->sL != nullptr && on;
}

void ensure_rows(gss_engine* e, int64_t V) {
  if (V <= e->cap_rows) return;
  GSS_CUDA(cudaDeviceSynchronize());
  const int64_t cap = std::min<int64_t>(e->n, std::max<int64_t>(V + V / 4, 1024));
  // The stage buffers hold live data across iterations (the pending gradients of g-1 feed
  // forward_params(g) and lazy(g-1)): grow them preserving their contents.
  auto grow = [&](float*& buf, int width) {
    float* nb = dmalloc<float>((size_t)cap * width);
    GSS_CUDA(cudaMemset(nb, 0, (size_t)cap * width * sizeof(float)));  // the copied tail is defined too
    if (buf) {
      GSS_CUDA(cudaMemcpy(nb, buf, (size_t)e->cap_rows * width * sizeof(float), cudaMemcpyDeviceToDevice));
      cudaFree(buf);
    }
    buf = nb;
  };
  for (int b = 0; b < 2; ++b) {
    grow(e->fwd[b], kNgDim);
    grow(e->g_geo[b], kGeoDim);
    grow(e->g_ng[b], kNgGradStride);
    grow(e->g_m2d[b], 2);
  }
  e->cap_rows = cap;
}

cudaEvent_t take_event(gss_engine* e) {
  if (!e->ev_free.empty()) {
    cudaEvent_t ev = e->ev_free.back();
    e->ev_free.pop_back();
    return ev;
  }
  cudaEvent_t ev;
  GSS_CUDA(cudaEventCreate(&ev));
  return ev;
}
constexpr int kTouchedRing = 64;
void stage_begin(gss_engine* e, int st, cudaStream_t s, int g, uint64_t bytes = 0, int touched_slot = -1) {
  nvtxRangePushA(kStageName[st]);
  if (!e->delays_ns.empty()) {
    stage_delay_kernel<<<1, 1, 0, s>>>(e->delays_ns[e->delay_next++ % e->delays_ns.size()]);
    GSS_LAUNCHED();
  }
  gss_engine::TimeRec r{st, take_event(e), take_event(e), g, (s == e->sH || s == e->sL) ? 1 : 0, bytes, touched_slot};
  GSS_CUDA(cudaEventRecord(r.a, s));
  e->pending_times.push_back(r);
}
void stage_end(gss_engine* e, int st, cudaStream_t s, int) {
  nvtxRangePop();
  for (auto it = e->pending_times.rbegin(); it != e->pending_times.rend(); ++it)
    if (it->stage == st) {
      GSS_CUDA(cudaEventRecord(it->b, s));
      return;
    }
}
void timeline_push(gss_engine* e, const gss_engine::TimeRec& r, const int64_t* touched_host) {
  if (!e->timeline_on || !e->epoch) return;
  float t0 = 0.0f, t1 = 0.0f;
  if (cudaEventElapsedTime(&t0, e->epoch, r.a) != cudaSuccess || cudaEventElapsedTime(&t1, e->epoch, r.b) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  gss_timeline_row row{};
  row.iteration = r.iter;
  row.stage = r.stage;
  row.worker = r.worker;
  row.t0_ns = (int64_t)((double)t0 * 1e6);
  row.t1_ns = (int64_t)((double)t1 * 1e6);
  row.bytes = r.bytes;
  if (r.touched_slot >= 0 && touched_host)  // adam.hpp:234-236: 7*dim*4 per touched row + 1 counter byte per row
    row.bytes = (uint64_t)touched_host[r.touched_slot] * 7u * kNgDim * 4u + (uint64_t)e->n;
  e->timeline.push_back(row);
}
// After a drain: fold the recorded stage intervals into stage_ms and recycle the events.
void collect_times(gss_engine* e) {
  int64_t touched[kTouchedRing] = {};
  if (e->timeline_on && e->touched_ring)
    GSS_CUDA(cudaMemcpy(touched, e->touched_ring, sizeof touched, cudaMemcpyDeviceToHost));
  for (auto& r : e->pending_times) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) e->stage_ms[r.stage] += ms;
    timeline_push(e, r, touched);
    e->ev_free.push_back(r.a);
    e->ev_free.push_back(r.b);
  }
  cudaGetLastError();
  e->pending_times.clear();
}
// Streaming (step()) without a drain: fold the intervals that have completed, so the event pool
// stays bounded however long the host streams steps between drains.
void collect_completed(gss_engine* e) {
  std::vector<gss_engine::TimeRec> keep;
  for (auto& r : e->pending_times) {
    if (cudaEventQuery(r.b) != cudaSuccess) {
      keep.push_back(r);
      continue;
    }
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) e->stage_ms[r.stage] += ms;
    timeline_push(e, r, nullptr);
    e->ev_free.push_back(r.a);
    e->ev_free.push_back(r.b);
  }
  cudaGetLastError();
  e->pending_times.swap(keep);
}

// Split-camera buffers sized for the current n (allocated on the first split camera; regrown
// after densification grows n — both streams are drained first, the plans in flight use them).
void ensure_split_buffers(gss_engine* e) {
  if (e->split_cap >= e->n && e->smask[0]) return;
  GSS_CUDA(cudaStreamSynchronize(e->sD));
  GSS_CUDA(cudaStreamSynchronize(e->sH));
  auto f = [](auto*& p) { if (p) cudaFree(p); p = nullptr; };
  const int64_t n = std::max<int64_t>(e->n, 1);
  const int64_t nwords = (n + 31) / 32;
  for (int k = 0; k < 2; ++k) {
    f(e->smask[k]);
    e->smask[k] = dmalloc<uint32_t>((size_t)nwords);
  }
  f(e->wpre);
  e->wpre = dmalloc<int32_t>((size_t)nwords + 1);
  for (int p = 0; p < 3; ++p)
    for (int k = 0; k < 2; ++k) {
      f(e->sids[p][k]);
      f(e->smap[p][k]);
      e->sids[p][k] = dmalloc<int32_t>((size_t)n);
      e->smap[p][k] = dmalloc<int32_t>((size_t)n);
      if (!e->scount[p][k]) e->scount[p][k] = dmalloc<int64_t>(1);
    }
  if (!e->scount_host) GSS_CUDA(cudaHostAlloc((void**)&e->scount_host, 6 * sizeof(int64_t), cudaHostAllocDefault));
  if (!e->sloss) e->sloss = dmalloc<float>(2);
  size_t tb = 0;
  GSS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, e->wpre, e->wpre, (int)(nwords + 1)));
  if (tb > e->scan_tmp_bytes) {
    f(e->scan_tmp);
    e->scan_tmp = dmalloc<char>(tb);
    e->scan_tmp_bytes = tb;
  }
  e->split_cap = n;
}

// Per-side gradient buffers of a split render (rows of the left / right sub-lists).
void ensure_split_rows(gss_engine* e, int64_t V) {
  if (V <= e->scap_rows) return;
  GSS_CUDA(cudaStreamSynchronize(e->sD));
  const int64_t cap = std::min<int64_t>(std::max<int64_t>(e->n, 1), std::max<int64_t>(V + V / 4, 1024));
  for (int k = 0; k < 2; ++k) {
    if (e->sg_geo[k]) cudaFree(e->sg_geo[k]);
    if (e->sg_ng[k]) cudaFree(e->sg_ng[k]);
    if (e->sg_m2d[k]) cudaFree(e->sg_m2d[k]);
    e->sg_geo[k] = dmalloc<float>((size_t)cap * kGeoDim);
    e->sg_ng[k] = dmalloc<float>((size_t)cap * kNgGradStride);
    e->sg_m2d[k] = dmalloc<float>((size_t)cap * 2);
  }
  e->scap_rows = cap;
}

int split_column_of(const gss_engine* e, int g, bool stored_camera) {
  if (!stored_camera || e->split_col.empty()) return -1;
  return e->split_col[(size_t)g % e->split_col.size()];
}

// engine.hpp:255-278. A split camera culls the left [0, column] and right [column, W] viewports
// (closed, as the reference's Viewport) and takes their sorted union; each side's slot map into
// the union feeds its render pass (engine.hpp:324-332).
void stage_cull(gss_engine* e, int g, const gss_camera& cam, int col) {
  const int p = g % 3;
  cudaStream_t s = e->sD;
  e->plan_col[p] = col;
  stage_begin(e, kCull, s, g, (uint64_t)e->n * 40u * (col >= 0 ? 2u : 1u));  // + 4 V for the ids (V not host-known yet)
  if (col < 0) {
    const gss_viewport vp{0.0f, (float)cam.width, 0.0f, (float)cam.height};
    cull(e->gw, e->n, kGeoDim, &cam, &vp, e->cfg.low_pass, nullptr, e->ids[p], e->count[p], e->cull_ws,
         e->cull_ws_bytes, s);
  } else {
    ensure_split_buffers(e);
    const gss_viewport lvp{0.0f, (float)col, 0.0f, (float)cam.height};
    const gss_viewport rvp{(float)col, (float)cam.width, 0.0f, (float)cam.height};
    cull(e->gw, e->n, kGeoDim, &cam, &lvp, e->cfg.low_pass, e->smask[0], e->sids[p][0], e->scount[p][0], e->cull_ws,
         e->cull_ws_bytes, s);
    cull(e->gw, e->n, kGeoDim, &cam, &rvp, e->cfg.low_pass, e->smask[1], e->sids[p][1], e->scount[p][1], e->cull_ws,
         e->cull_ws_bytes, s);
    const int64_t nwords = (e->n + 31) / 32;
    union_popc_kernel<<<(unsigned)ceil_div(nwords + 1, 256), 256, 0, s>>>(e->smask[0], e->smask[1], nwords, e->wpre);
    GSS_LAUNCHED();
    size_t tb = e->scan_tmp_bytes;
    GSS_CUDA(cub::DeviceScan::ExclusiveSum(e->scan_tmp, tb, e->wpre, e->wpre, (int)(nwords + 1), s));
    union_ids_kernel<<<(unsigned)ceil_div(nwords + 1, 256), 256, 0, s>>>(e->smask[0], e->smask[1], e->wpre, nwords,
                                                                         e->ids[p], e->count[p]);
    GSS_LAUNCHED();
    for (int k = 0; k < 2; ++k) {
      union_slot_kernel<<<148 * 8, 256, 0, s>>>(e->sids[p][k], e->scount[p][k], e->smask[0], e->smask[1], e->wpre,
                                                e->smap[p][k]);
      GSS_LAUNCHED();
      GSS_CUDA(cudaMemcpyAsync(e->scount_host + 2 * p + k, e->scount[p][k], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
  }
  GSS_CUDA(cudaMemcpyAsync(e->count_host + p, e->count[p], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  stage_end(e, kCull, s, g & 1);
  GSS_CUDA(cudaEventRecord(e->ev_cull[p].e, s));
}

// engine.hpp:282-307: restore_view of ids(g) with pending grads(g-1).
void stage_forward_params(gss_engine* e, int g) {
  const int p = g % 3, b = g % 2;
  cudaStream_t s = S(e, true);
  const bool conc = host_concurrent(e);
  if (e->cfg.pipelined) {
    GSS_CUDA(cudaStreamWaitEvent(s, e->ev_cull[p].e, 0));
    if (g > e->seg_begin) GSS_CUDA(cudaStreamWaitEvent(s, e->ev_handoff[(g - 1) % 2].e, 0));
    // fwd[b] is free once render(g-2) consumed it
    GSS_CUDA(cudaStreamWaitEvent(s, e->ev_render[b].e, 0));
    // concurrent host tier: the lazy updates run on sL; fp(g) reads the state after lazy(g-2)
    if (conc) GSS_CUDA(cudaStreamWaitEvent(s, e->ev_lazy[b].e, 0));
  }
  // V is needed on the host to size staging buffers: wait for this plan's count.
  GSS_CUDA(cudaEventSynchronize(e->ev_cull[p].e));
  const int64_t V = e->count_host[p];
  ensure_rows(e, V);
  const int pb = (g - 1) % 2;
  const bool pending = g > e->seg_begin && e->g_iter[pb] == g - 1;
  // V (3*196 + 1) + V_pend * 196 + V * 196
  const uint64_t fbytes = (uint64_t)V * (3 * 196 + 1 + 196) +
                          (pending ? (uint64_t)e->count_host[e->g_plan[pb]] * 196u : 0u);
  stage_begin(e, kFwd, s, g, fbytes);
  gss_sparse_grads pg{};
  if (pending) {
    const int pp = e->g_plan[pb];
    pg.ids = e->ids[pp];
    pg.count = e->count_host[pp];
    pg.count_dev = e->count[pp];
    pg.rows = e->g_ng[pb];
    pg.stride = kNgGradStride;
    pg.col0 = 0;
  }
  // (the host tier takes the host-known count: its gather is staged through HBM in one pass)
  adam_restore(&e->ng, e->ids[p], V, e->ng_host ? nullptr : e->count[p], pending ? &pg : nullptr, e->fwd[b], s,
               conc ? e->ev_resolved[b].e : nullptr);
  e->fwd_iter[b] = g;
  stage_end(e, kFwd, s, b);
  GSS_CUDA(cudaEventRecord(e->ev_fp[b].e, s));
}

// engine.hpp:311-377.
void stage_render(gss_engine* e, int g, const gss_camera& cam, const float* gt_dev, float* loss_out) {
  const int p = g % 3, b = g % 2;
  cudaStream_t s = e->sD;
  require(e->fwd_iter[b] == g, "render: forwarded buffer is not for this iteration", GSS_ERR_INVARIANT);
  stage_begin(e, kRender, s, g);
  const int64_t V = e->count_host[p];
  gss_render_scene sc{};
  sc.ids = e->ids[p];
  sc.count = V;
  sc.geo = e->gw;
  sc.geo_stride = kGeoDim;
  sc.nongeo = e->fwd[b];
  sc.nongeo_stride = kNgDim;
  sc.nongeo_compact = 1;
  const int deg = e->cfg.sh_warmup_step > 0 ? std::min(e->cfg.sh_degree, g / e->cfg.sh_warmup_step)
                                            : e->cfg.sh_degree;  // engine.hpp:45-48
  sc.sh_degree = deg;
  for (int c = 0; c < 3; ++c) sc.background[c] = e->cfg.background[c];
  sc.low_pass = e->cfg.low_pass;
  const int64_t full = (int64_t)cam.width * cam.height * 3;
  const int col = e->plan_col[p];
  // The waits of the composite: fp(g) (pipelined), the gradient stage's previous reader, and the
  // step's ground-truth copy.
  // step(): the ground truth was copied in on sC, overlapping cull/geometry/gather
  const bool step_gt = e->gt_pending;
  e->gt_pending = false;
  bool waited = false;
  auto wait_inputs = [&] {
    if (waited) return;
    waited = true;
    if (e->cfg.pipelined) {
      GSS_CUDA(cudaStreamWaitEvent(s, e->ev_fp[b].e, 0));
      // grads[b] is free once lazy(g-2) consumed it
      GSS_CUDA(cudaStreamWaitEvent(s, e->ev_lazy[b].e, 0));
    }
    if (step_gt) GSS_CUDA(cudaStreamWaitEvent(s, e->ev_gt.e, 0));
  };
  if (col < 0) {
    const gss_viewport vp{0.0f, (float)cam.width, 0.0f, (float)cam.height};
    // Geometry half first: it reads only the geometric tier, so in pipelined mode it overlaps the
    // forwarding gather of this iteration on stream H; colour + composite wait for fp(g).
    rasterize_forward_geometry(e->rctx, &sc, &cam, &vp, s);
    wait_inputs();
    rasterize_forward_finish(e->rctx, e->image, gt_dev, full, e->d_img, loss_out, s);
    rasterize_backward(e->rctx, e->d_img, e->g_geo[b], kGeoDim, e->g_ng[b], kNgGradStride, e->g_m2d[b], s);
  } else {
    // engine.hpp:355-371: two sub-passes (left, right viewport), each normalised by the full image,
    // loss = ll + rl, gradients aggregated over the union (left added first).
    ensure_split_rows(e, std::max(e->scount_host[2 * p], e->scount_host[2 * p + 1]));
    for (int k = 0; k < 2; ++k) {
      gss_render_scene ss = sc;
      ss.ids = e->sids[p][k];
      ss.count = e->scount_host[2 * p + k];
      ss.slot_map = e->smap[p][k];
      const gss_viewport vp = k == 0 ? gss_viewport{0.0f, (float)col, 0.0f, (float)cam.height}
                                     : gss_viewport{(float)col, (float)cam.width, 0.0f, (float)cam.height};
      rasterize_forward_geometry(e->rctx, &ss, &cam, &vp, s);
      wait_inputs();
      rasterize_forward_finish(e->rctx, e->image, gt_dev, full, e->d_img, e->sloss + k, s);
      rasterize_backward(e->rctx, e->d_img, e->sg_geo[k], kGeoDim, e->sg_ng[k], kNgGradStride, e->sg_m2d[k], s);
    }
    GSS_CUDA(cudaMemsetAsync(e->g_geo[b], 0, (size_t)V * kGeoDim * 4, s));
    GSS_CUDA(cudaMemsetAsync(e->g_ng[b], 0, (size_t)V * kNgGradStride * 4, s));
    GSS_CUDA(cudaMemsetAsync(e->g_m2d[b], 0, (size_t)V * 2 * 4, s));
    for (int k = 0; k < 2; ++k) {
      const int64_t* cnt = e->scount[p][k];
      const int32_t* map = e->smap[p][k];
      add_rows_kernel<<<148 * 8, 256, 0, s>>>(e->sg_geo[k], kGeoDim, map, cnt, kGeoDim, e->g_geo[b]);
      GSS_LAUNCHED();
      add_rows_kernel<<<148 * 8, 256, 0, s>>>(e->sg_ng[k], kNgGradStride, map, cnt, kNgDim, e->g_ng[b]);
      GSS_LAUNCHED();
      add_rows_kernel<<<148 * 8, 256, 0, s>>>(e->sg_m2d[k], 2, map, cnt, 2, e->g_m2d[b]);
      GSS_LAUNCHED();
    }
    split_loss_kernel<<<1, 1, 0, s>>>(e->sloss, loss_out);
    GSS_LAUNCHED();
  }
  if (step_gt) GSS_CUDA(cudaEventRecord(e->ev_gt_done[e->gt_cur].e, s));  // its buffer is free again
  e->g_plan[b] = p;
  stage_end(e, kRender, s, b);
  GSS_CUDA(cudaEventRecord(e->ev_render[b].e, s));
}

// engine.hpp:380-386: immediate dense update of the geometric tier (geo_defer_max = 0).
void stage_geo_update(gss_engine* e, int g) {
  const int p = g % 3, b = g % 2;
  cudaStream_t s = e->sD;
  stage_begin(e, kGeo, s, g, (uint64_t)e->n * 240u + (uint64_t)e->count_host[p] * 40u);
  gss_sparse_grads gr{};
  gr.ids = e->ids[p];
  gr.count = e->count_host[p];
  gr.count_dev = e->count[p];
  gr.rows = e->g_geo[b];
  gr.stride = kGeoDim;
  gr.col0 = 0;
  adam_update(&e->geo, &gr, nullptr, nullptr, s);
  stage_end(e, kGeo, s, b);
}

// engine.hpp:391-417: gradients stay in HBM (the stage buffer render wrote); densification
// statistics are accumulated and the stage is handed to forward_params(g+1) / lazy(g).
void stage_handoff(gss_engine* e, int g) {
  const int p = g % 3, b = g % 2;
  cudaStream_t s = e->sD;
  stage_begin(e, kHandoff, s, g, (uint64_t)e->count_host[p] * (8u + 12u + 8u + 4u));
  const int64_t V = e->count_host[p];
  if (V > 0) {
    const int blocks = (int)std::min<int64_t>(ceil_div(V, 256), 148 * 8);
    handoff_stats_kernel<<<blocks, 256, 0, s>>>(e->ids[p], e->count[p], e->g_m2d[b], e->accum_norm, e->accum_cnt);
    GSS_LAUNCHED();
  }
  e->g_iter[b] = g;
  stage_end(e, kHandoff, s, b);
  GSS_CUDA(cudaEventRecord(e->ev_handoff[b].e, s));
}

// engine.hpp:420-430: lazy deferred update of the non-geometric tier with grads(g).
// Concurrent host tier (next >= 0: fp(next) is in flight on stream H): on stream sL, after fp(next)'s
// resolve pass has read the counters, pass 1 updates them; the walk of the touched rows outside
// ids(next) runs beside fp(next)'s gather (disjoint rows), and the walk of the touched rows inside
// ids(next) waits for that gather (it must read them before they are updated) — the reference's
// order fp(next) -> lazy(g) for every row both touch, with the link's two directions busy at once.
void stage_lazy(gss_engine* e, int g, int next = -1) {
  const int b = g % 2;
  const bool conc = host_concurrent(e);
  cudaStream_t s = conc ? e->sL : S(e, true);
  require(e->g_iter[b] == g, "lazy update: staging buffer holds a different iteration", GSS_ERR_INVARIANT);
  if (e->cfg.pipelined) GSS_CUDA(cudaStreamWaitEvent(s, e->ev_handoff[b].e, 0));
  const int pn = next >= 0 ? next % 3 : -1;
  if (conc && next >= 0) {
    GSS_CUDA(cudaStreamWaitEvent(s, e->ev_resolved[next % 2].e, 0));
    mark_rows_kernel<<<148 * 4, 256, 0, s>>>(e->ids[pn], e->count[pn], e->vis_mask, 1);
    GSS_LAUNCHED();
  }
  const int slot = e->timeline_on ? (e->touched_next++ % kTouchedRing) : -1;
  stage_begin(e, kLazy, s, g, 0, slot);
  const int p = e->g_plan[b];
  gss_sparse_grads gr{};
  gr.ids = e->ids[p];
  gr.count = e->count_host[p];
  gr.count_dev = e->count[p];
  gr.rows = e->g_ng[b];
  gr.stride = kNgGradStride;
  gr.col0 = 0;
  if (e->ng_host) set_host_chunk_bytes(e->cfg.chunk_bytes);  // staged host-tier chunks (store.hpp:204-213)
  if (conc && next >= 0) {
    adam_update(&e->ng, &gr, nullptr, slot >= 0 ? e->touched_ring + slot : nullptr, s, e->vis_mask,
                e->ev_fp[next % 2].e);
    mark_rows_kernel<<<148 * 4, 256, 0, s>>>(e->ids[pn], e->count[pn], e->vis_mask, 0);
    GSS_LAUNCHED();
  } else {
    adam_update(&e->ng, &gr, nullptr, slot >= 0 ? e->touched_ring + slot : nullptr, s);
  }
  stage_end(e, kLazy, s, b);
  GSS_CUDA(cudaEventRecord(e->ev_lazy[b].e, s));
}

// One iteration g of the DAG. Serial mode keeps run_serial's order on one stream
// (engine.hpp:434-445); pipelined mode enqueues lazy(g-1) on the host-tier stream right after
// fp(g) so it overlaps render(g) (engine.hpp:498-508). The data each stage reads is the same in
// both orders, so the trajectories are bitwise identical.
void iteration(gss_engine* e, int g, const gss_camera& cam, const float* gt_dev, float* loss_out, int col = -1) {
  nvtxRangePushA("iteration");
  stage_cull(e, g, cam, col);
  stage_forward_params(e, g);
  const int owed = e->open_pending;
  // lazy(g-1) runs on stream H after fp(g) in both modes (pipelined: overlapping render(g) on D;
  // the concurrent host tier: on stream sL, partly beside fp(g)). It is enqueued after render(g): a
  // staged host-tier pass reads its touched count back before chunking (staged_walk), and render(g)
  // must already be queued on D by then.
  stage_render(e, g, cam, gt_dev, loss_out);
  if (owed >= 0) stage_lazy(e, owed, g);
  stage_geo_update(e, g);
  stage_handoff(e, g);
  e->open_pending = g;
  e->valid_counts.push_back(e->count_host[g % 3]);
  nvtxRangePop();
}

void drain(gss_engine* e) {
  if (e->open_pending >= 0) {
    stage_lazy(e, e->open_pending);
    e->open_pending = -1;
  }
  GSS_CUDA(cudaStreamSynchronize(e->sD));
  GSS_CUDA(cudaStreamSynchronize(e->sH));
  if (e->sL) GSS_CUDA(cudaStreamSynchronize(e->sL));
  collect_times(e);
}

void ensure_loss(gss_engine* e, int n) {
  if (n <= e->loss_cap) return;
  GSS_CUDA(cudaDeviceSynchronize());
  cudaFree(e->loss_dev);
  e->loss_dev = dmalloc<float>((size_t)n);
  e->loss_cap = n;
}

void setup_arena(gss_arena& a, float* w, float* m, float* v, uint8_t* c, int64_t n, int dim, int defer_max,
                 bool geo, const gss_engine_config& cfg) {
  a = gss_arena{};
  a.w = w; a.m = m; a.v = v; a.counter = c; a.n = n; a.dim = dim; a.defer_max = defer_max; a.step = 0;
  auto grp = [&](int col0, int d, double lr) {
    gss_group gg{col0, d, lr, cfg.beta1, cfg.beta2, cfg.eps};
    a.groups[a.ngroups++] = gg;
  };
  if (geo) {  // store.hpp:129-131
    grp(0, 3, cfg.lr_mean * cfg.scene_extent);
    grp(3, 3, cfg.lr_scale);
    grp(6, 4, cfg.lr_quat);
  } else {  // store.hpp:132-136
    grp(0, 1, cfg.lr_opacity);
    grp(1, 3, cfg.lr_sh);
    grp(4, 45, cfg.lr_sh / cfg.sh_rest_divisor);
  }
}

}  // namespace

void engine_config_default(gss_engine_config* c) {
  *c = gss_engine_config{};
  c->lr_mean = 1.6e-4; c->lr_scale = 5e-3; c->lr_quat = 1e-3; c->lr_opacity = 5e-2; c->lr_sh = 2.5e-3;
  c->sh_rest_divisor = 20.0; c->beta1 = 0.9; c->beta2 = 0.999; c->eps = 1e-8; c->scene_extent = 1.0;
  c->defer_max = 15; c->geo_defer_max = 0; c->pipelined = 1; c->sh_degree = 3; c->sh_warmup_step = 0;
  c->background[0] = c->background[1] = c->background[2] = 0.0f;
  c->low_pass = 0.3f;
  c->nongeo_on_host = 0;
  c->chunk_bytes = int64_t(32) << 20;
}

gss_engine* engine_create(int64_t n, const float* rows, int32_t ncams, const gss_camera* cams, const float* gts,
                          const gss_engine_config* cfg) {
  require(n >= 0 && n <= INT32_MAX, "engine: n out of range");
  require(n == 0 || rows, "engine: null init rows");
  require(ncams >= 0 && (ncams == 0 || cams), "engine: null cameras");
  require(cfg != nullptr, "engine: null config");
  require(cfg->defer_max >= 0 && cfg->defer_max <= 254 && cfg->geo_defer_max >= 0 && cfg->geo_defer_max <= 254,
          "config: defer max must be in [0,254]");
  require(cfg->sh_degree >= 0 && cfg->sh_degree <= 3, "config: sh_degree must be in [0,3]");
  for (int i = 0; i < ncams; ++i) {
    require(cams[i].near_plane > 0 && cams[i].far_plane > cams[i].near_plane, "camera: require 0 < near < far");
    require(cams[i].width >= 1 && cams[i].height >= 1, "camera: require W, H >= 1");
  }
  auto e = std::make_unique<gss_engine>();
  e->cfg = *cfg;
  e->n = n;
  e->cams.assign(cams, cams + ncams);
  e->ng_host = cfg->nongeo_on_host != 0;
  {
    // Stream priorities (GSS_STREAM_PRIO, A/B): 0 = equal, 1 = stream H first (its link-bound
    // host-tier passes get their few CTAs scheduled ahead of the render), 2 = stream D first
    // (the render's geometry phase, on the critical path, is not slowed by the concurrent
    // forwarding gather / lazy update).
    int lo = 0, hi = 0;
    GSS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char* ev = std::getenv("GSS_STREAM_PRIO");
    // default 1: measured equal to 0 within noise at C4 and ahead of 2 (which starves the lazy
    // update behind the render: profiles/r02_stream_priority_ab.txt)
    const int mode = ev ? std::atoi(ev) : 1;
    GSS_CUDA(cudaStreamCreateWithPriority(&e->sD, cudaStreamNonBlocking, mode == 2 ? hi : lo));
    GSS_CUDA(cudaStreamCreateWithPriority(&e->sH, cudaStreamNonBlocking, mode == 1 ? hi : lo));
    if (e->ng_host) GSS_CUDA(cudaStreamCreateWithPriority(&e->sL, cudaStreamNonBlocking, mode == 1 ? hi : lo));
  }
  GSS_CUDA(cudaStreamCreateWithFlags(&e->sC, cudaStreamNonBlocking));
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  e->gw = dmalloc<float>(nn * kGeoDim);
  e->gm = dmalloc<float>(nn * kGeoDim);
  e->gv = dmalloc<float>(nn * kGeoDim);
  e->gcnt = dmalloc<uint8_t>(nn);
  // The host tier's w/m/v live in pinned host memory; its counters (1 byte per row, read and
  // written by the device passes only) stay in HBM.
  if (e->ng_host)
    GSS_CUDA(cudaHostAlloc((void**)&e->nw, nn * kNgStride * 4, cudaHostAllocMapped));
  else
    e->nw = dmalloc<float>(nn * kNgStride);
  e->ncnt = dmalloc<uint8_t>(nn);
  if (e->ng_host) {
    e->vis_mask = dmalloc<uint32_t>((nn + 31) / 32);
    GSS_CUDA(cudaMemsetAsync(e->vis_mask, 0, (nn + 31) / 32 * 4, e->sD));
  }
  e->nm = e->nw + kNgSeg;
  e->nv = e->nw + 2 * kNgSeg;
  GSS_CUDA(cudaMemsetAsync(e->gm, 0, nn * kGeoDim * 4, e->sD));
  GSS_CUDA(cudaMemsetAsync(e->gv, 0, nn * kGeoDim * 4, e->sD));
  GSS_CUDA(cudaMemsetAsync(e->gcnt, 0, nn, e->sD));
  GSS_CUDA(cudaMemsetAsync(e->nw, 0, nn * kNgStride * 4, e->sD));
  GSS_CUDA(cudaMemsetAsync(e->ncnt, 0, nn, e->sD));
  if (n > 0) {
    float* rows_dev = dmalloc<float>((size_t)n * kRowDim);
    GSS_CUDA(cudaMemcpyAsync(rows_dev, rows, (size_t)n * kRowDim * 4, cudaMemcpyHostToDevice, e->sD));
    split_rows_kernel<<<(unsigned)ceil_div(n * kRowDim, 256), 256, 0, e->sD>>>(rows_dev, n, e->gw, e->nw);
    GSS_LAUNCHED();
    GSS_CUDA(cudaStreamSynchronize(e->sD));
    cudaFree(rows_dev);
  }
  setup_arena(e->geo, e->gw, e->gm, e->gv, e->gcnt, n, kGeoDim, cfg->geo_defer_max, true, *cfg);
  setup_arena(e->ng, e->nw, e->nm, e->nv, e->ncnt, n, kNgDim, cfg->defer_max, false, *cfg);
  e->ng.row_stride = kNgStride;
  for (int p = 0; p < 3; ++p) {
    e->ids[p] = dmalloc<int32_t>(nn);
    e->count[p] = dmalloc<int64_t>(1);
  }
  GSS_CUDA(cudaHostAlloc((void**)&e->count_host, 3 * sizeof(int64_t), cudaHostAllocDefault));
  e->cull_ws_bytes = cull_workspace_bytes(n);
  e->cull_ws = dmalloc<char>(e->cull_ws_bytes);
  GSS_CUDA(cudaMemsetAsync(e->cull_ws, 0, e->cull_ws_bytes, e->sD));  // zero once (gss_cull contract)
  e->accum_norm = dmalloc<double>(nn);
  e->accum_cnt = dmalloc<int32_t>(nn);
  GSS_CUDA(cudaMemsetAsync(e->accum_norm, 0, nn * 8, e->sD));
  GSS_CUDA(cudaMemsetAsync(e->accum_cnt, 0, nn * 4, e->sD));
  int maxW = 1, maxH = 1;
  for (const auto& c : e->cams) {
    maxW = std::max(maxW, c.width);
    maxH = std::max(maxH, c.height);
  }
  e->W = maxW;
  e->H = maxH;
  const size_t img = (size_t)maxW * maxH * 3;
  e->image = dmalloc<float>(img);
  e->d_img = dmalloc<float>(img);
  e->gt_step[0] = dmalloc<float>(img);
  e->gt_step[1] = dmalloc<float>(img);
  if (gts && ncams > 0) {
    e->gts_dev = dmalloc<float>(img * ncams);
    size_t off = 0;
    for (int i = 0; i < ncams; ++i) {
      const size_t sz = (size_t)cams[i].width * cams[i].height * 3;
      GSS_CUDA(cudaMemcpyAsync(e->gts_dev + img * i, gts + off, sz * 4, cudaMemcpyHostToDevice, e->sD));
      off += sz;
    }
  }
  e->rctx = render_ctx_create();
  // Reserve every per-view buffer for the stored cameras: each is culled and rendered once (forward
  // + backward with a zero image gradient; no optimizer state changes), so the stage buffers and
  // the rasterizer's records, sort keys, instance partials and per-pixel buffers reach their size
  // before run() — its first visit of a larger view does not stop to grow them. Later growth (the
  // scene moves, densification) still happens on demand.
  if (n > 0 && !e->cams.empty()) {
    int64_t vmax = 0;
    GSS_CUDA(cudaMemsetAsync(e->d_img, 0, (size_t)e->W * e->H * 3 * sizeof(float), e->sD));
    for (const auto& c : e->cams) {
      const gss_viewport vp{0.0f, (float)c.width, 0.0f, (float)c.height};
      cull(e->gw, e->n, kGeoDim, &c, &vp, cfg->low_pass, nullptr, e->ids[0], e->count[0], e->cull_ws,
           e->cull_ws_bytes, e->sD);
      GSS_CUDA(cudaMemcpyAsync(e->count_host, e->count[0], sizeof(int64_t), cudaMemcpyDeviceToHost, e->sD));
      GSS_CUDA(cudaStreamSynchronize(e->sD));
      const int64_t V = e->count_host[0];
      vmax = std::max(vmax, V);
      ensure_rows(e.get(), std::min<int64_t>(n, vmax + vmax / 4));
      gss_render_scene sc{};
      sc.ids = e->ids[0];
      sc.count = V;
      sc.geo = e->gw;
      sc.geo_stride = kGeoDim;
      sc.nongeo = e->nw;  // the stored rows by id (w segment of the interleaved tier)
      sc.nongeo_stride = kNgStride;
      sc.nongeo_compact = 0;
      sc.sh_degree = cfg->sh_degree;
      sc.low_pass = cfg->low_pass;
      rasterize_forward_geometry(e->rctx, &sc, &c, &vp, e->sD);
      rasterize_forward_finish(e->rctx, e->image, nullptr, 0, nullptr, nullptr, e->sD);
      rasterize_backward(e->rctx, e->d_img, e->g_geo[0], kGeoDim, e->g_ng[0], kNgGradStride, e->g_m2d[0], e->sD);
    }
  }
  GSS_CUDA(cudaStreamSynchronize(e->sD));
  return e.release();
}

void engine_destroy(gss_engine* e) {
  if (!e) return;
  cudaDeviceSynchronize();
  try {
    arena_release(&e->geo);
    arena_release(&e->ng);
  } catch (...) {
  }
  auto f = [](void* p) { if (p) cudaFree(p); };
  f(e->gts_dev); f(e->gw); f(e->gm); f(e->gv); f(e->gcnt);
  if (e->ng_host) cudaFreeHost(e->nw); else f(e->nw);
  f(e->ncnt);
  for (int p = 0; p < 3; ++p) { f(e->ids[p]); f(e->count[p]); }
  if (e->count_host) cudaFreeHost(e->count_host);
  f(e->cull_ws);
  for (int b = 0; b < 2; ++b) { f(e->fwd[b]); f(e->g_geo[b]); f(e->g_ng[b]); f(e->g_m2d[b]); }
  render_ctx_destroy(e->rctx);
  f(e->image); f(e->d_img); f(e->gt_step[0]); f(e->gt_step[1]); f(e->loss_dev); f(e->accum_norm); f(e->accum_cnt);
  e->timeline_on = false;
  collect_times(e);
  for (auto ev : e->ev_free) cudaEventDestroy(ev);
  if (e->epoch) cudaEventDestroy(e->epoch);
  f(e->touched_ring);
  for (int k = 0; k < 2; ++k) { f(e->smask[k]); f(e->sg_geo[k]); f(e->sg_ng[k]); f(e->sg_m2d[k]); }
  for (int p = 0; p < 3; ++p)
    for (int k = 0; k < 2; ++k) { f(e->sids[p][k]); f(e->smap[p][k]); f(e->scount[p][k]); }
  f(e->wpre); f(e->scan_tmp); f(e->sloss);
  if (e->scount_host) cudaFreeHost(e->scount_host);
  if (e->sD) cudaStreamDestroy(e->sD);
  if (e->sH) cudaStreamDestroy(e->sH);
  if (e->sC) cudaStreamDestroy(e->sC);
  if (e->sL) cudaStreamDestroy(e->sL);
  f(e->vis_mask);
  cudaGetLastError();
  delete e;
}

// OffloadEngine::run (engine.hpp:73-88): n iterations over the stored cameras, then drained.
void engine_run(gss_engine* e, int iters, float* losses, int32_t* valid) {
  require(e != nullptr, "engine: null");
  require(iters >= 0, "engine: negative iteration count");
  if (iters == 0) return;
  require(!e->cams.empty(), "engine: no cameras");
  require(e->gts_dev != nullptr, "engine: run() needs stored ground-truth images");
  require(e->open_pending < 0, "engine: run() inside an open step() segment; call drain first",
          GSS_ERR_INVARIANT);
  const int64_t l0 = launches();
  ensure_loss(e, iters);
  const int g0 = e->next_iter;
  e->seg_begin = g0;
  e->valid_counts.clear();
  const size_t img = (size_t)e->W * e->H * 3;
  for (int j = 0; j < iters; ++j) {
    const int g = g0 + j;
    const size_t ci = (size_t)g % e->cams.size();
    iteration(e, g, e->cams[ci], e->gts_dev + img * ci, e->loss_dev + j, split_column_of(e, g, true));
  }
  drain(e);
  e->next_iter = g0 + iters;
  if (losses) GSS_CUDA(cudaMemcpy(losses, e->loss_dev, (size_t)iters * 4, cudaMemcpyDeviceToHost));
  if (valid)
    for (int j = 0; j < iters; ++j) valid[j] = (int32_t)e->valid_counts[j];
  e->launches_last = launches() - l0;
}

// Streaming entry point: one iteration with a host camera + ground truth. The segment stays open
// (the lazy update of this iteration is applied by the next step, exactly as inside run()).
// Synchronous: returns this step's loss. Asynchronous (wait = false): returns after enqueueing; the
// loss lands in *loss_host (pinned) when the iteration's render is done (gss_engine_drain waits), so
// the host prepares step g+1 — and its ground-truth copy — while step g still renders.
void engine_step(gss_engine* e, const gss_camera* cam, const float* gt_host, float* loss_host, int32_t* valid_host,
                 bool wait) {
  require(e && cam && gt_host, "engine_step: null argument");
  require(cam->width <= e->W && cam->height <= e->H, "engine_step: camera larger than the engine's image buffers");
  require(cam->near_plane > 0 && cam->far_plane > cam->near_plane, "camera: require 0 < near < far");
  require(wait || loss_host, "engine_step: an asynchronous step needs a (pinned) loss destination");
  const int64_t l0 = launches();
  ensure_loss(e, 1);
  if (e->pending_times.size() > 512) collect_completed(e);
  const int g = e->next_iter;
  if (e->open_pending < 0) {
    e->seg_begin = g;
    e->valid_counts.clear();
  }
  const size_t bytes = (size_t)cam->width * cam->height * 3 * 4;
  // Double-buffered ground truth: buffer gb is free once the composite of step g-2 (its last reader)
  // is done; the copy runs on its own stream and only this step's composite waits for it.
  const int gb = g & 1;
  GSS_CUDA(cudaStreamWaitEvent(e->sC, e->ev_gt_done[gb].e, 0));
  GSS_CUDA(cudaMemcpyAsync(e->gt_step[gb], gt_host, bytes, cudaMemcpyHostToDevice, e->sC));
  GSS_CUDA(cudaEventRecord(e->ev_gt.e, e->sC));
  e->gt_pending = true;
  e->gt_cur = gb;
  iteration(e, g, *cam, e->gt_step[gb], e->loss_dev);
  e->next_iter = g + 1;
  if (valid_host) *valid_host = (int32_t)e->count_host[g % 3];
  if (wait) {
    float l = 0.0f;
    GSS_CUDA(cudaMemcpyAsync(&l, e->loss_dev, 4, cudaMemcpyDeviceToHost, e->sD));
    GSS_CUDA(cudaStreamSynchronize(e->sD));
    if (loss_host) *loss_host = l;
  } else {
    GSS_CUDA(cudaMemcpyAsync(loss_host, e->loss_dev, 4, cudaMemcpyDeviceToHost, e->sD));
  }
  e->launches_last = launches() - l0;
}

// SplitTable (splitter.hpp:12-23) given to the OffloadEngine constructor (engine.hpp:62-68): per
// stored camera a split flag and column s in (0, W). Applies to run(); step() renders whole views.
void engine_set_splits(gss_engine* e, int32_t ncams, const int32_t* split, const int32_t* column) {
  require(e != nullptr, "engine: null");
  require(e->open_pending < 0, "engine: set_splits inside an open step() segment; call drain first",
          GSS_ERR_INVARIANT);
  if (ncams == 0) {
    e->split_col.clear();
    return;
  }
  require(split && column, "engine: null split table");
  require((size_t)ncams == e->cams.size(), "engine: split table size differs from the camera count");
  std::vector<int32_t> cols((size_t)ncams, -1);
  for (int i = 0; i < ncams; ++i) {
    if (!split[i]) continue;
    require(column[i] > 0 && column[i] < e->cams[i].width, "engine: split column must lie in (0, W)");
    cols[i] = column[i];
  }
  e->split_col = cols;
}

void engine_drain(gss_engine* e) {
  require(e != nullptr, "engine: null");
  drain(e);
}

namespace {
// Restored parameters of both tiers joined to n x 59 rows in device memory (engine.hpp:91-111).
float* snapshot_dev(gss_engine* e, cudaStream_t s) {
  const int64_t n = e->n;
  int32_t* all = dmalloc<int32_t>((size_t)n);
  float* geo = dmalloc<float>((size_t)n * kGeoDim);
  float* ng = dmalloc<float>((size_t)n * kNgDim);
  float* rows = dmalloc<float>((size_t)n * kRowDim);
  iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(all, n);
  GSS_LAUNCHED();
  adam_restore(&e->geo, all, n, nullptr, nullptr, geo, s);
  adam_restore(&e->ng, all, n, nullptr, nullptr, ng, s);
  join_rows_kernel<<<(unsigned)ceil_div(n * kRowDim, 256), 256, 0, s>>>(geo, ng, n, rows);
  GSS_LAUNCHED();
  GSS_CUDA(cudaStreamSynchronize(s));
  cudaFree(all); cudaFree(geo); cudaFree(ng);
  return rows;
}

// apply_densify (engine.hpp:116-163): row j < nsurv of the new tiers = old row survivors[j] (stored
// w/m/v and counter); row nsurv + k = child k (w from the child row, zero state).
__global__ void densify_apply_kernel(int64_t nsurv, int64_t nchild, const int32_t* survivors, const float* children,
                                     const float* gw, const float* gm, const float* gv, const uint8_t* gc,
                                     const float* nwold, const uint8_t* nc, float* gw2, float* gm2, float* gv2,
                                     uint8_t* gc2, float* nw2, uint8_t* nc2) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nsurv + nchild) return;
  if (j < nsurv) {
    const int64_t o = survivors[j];
    for (int c = 0; c < kGeoDim; ++c) {
      gw2[j * kGeoDim + c] = gw[o * kGeoDim + c];
      gm2[j * kGeoDim + c] = gm[o * kGeoDim + c];
      gv2[j * kGeoDim + c] = gv[o * kGeoDim + c];
    }
    for (int c = 0; c < kNgStride; ++c) nw2[j * kNgStride + c] = nwold[o * kNgStride + c];  // w, m, v
    gc2[j] = gc[o];
    nc2[j] = nc[o];
  } else {
    const float* row = children + (j - nsurv) * kRowDim;
    for (int c = 0; c < kGeoDim; ++c) {
      gw2[j * kGeoDim + c] = row[c];
      gm2[j * kGeoDim + c] = 0.0f;
      gv2[j * kGeoDim + c] = 0.0f;
    }
    for (int c = 0; c < kNgStride; ++c) nw2[j * kNgStride + c] = 0.0f;
    for (int c = 0; c < kNgDim; ++c) nw2[j * kNgStride + c] = row[kGeoDim + c];
    gc2[j] = 0;
    nc2[j] = 0;
  }
}
}  // namespace

// snapshot (engine.hpp:91-111): both tiers restored (no pending pass), joined to n x 59.
void engine_snapshot(gss_engine* e, float* rows_out) {
  require(e && rows_out, "snapshot: null argument");
  if (e->open_pending >= 0) drain(e);
  const int64_t n = e->n;
  if (n == 0) return;
  cudaStream_t s = e->sD;
  float* rows = snapshot_dev(e, s);
  GSS_CUDA(cudaMemcpy(rows_out, rows, (size_t)n * kRowDim * 4, cudaMemcpyDeviceToHost));
  cudaFree(rows);
}

// Densification event (trainer.hpp:578-591 with engine.hpp:116-163): snapshot, plan_densify on the
// device statistics, apply. counts[0..5] = survivors, children, clones, splits, pruned, new n.
void engine_densify(gss_engine* e, const gss_densify_config* dc, double extent, uint64_t seed, int64_t* counts) {
  require(e && dc && counts, "densify: null argument");
  if (e->open_pending >= 0) drain(e);
  GSS_CUDA(cudaDeviceSynchronize());
  cudaStream_t s = e->sD;
  const int64_t n = e->n;
  float* rows = n > 0 ? snapshot_dev(e, s) : nullptr;
  int32_t* surv = dmalloc<int32_t>((size_t)std::max<int64_t>(n, 1));
  float* children = dmalloc<float>((size_t)std::max<int64_t>(2 * n, 1) * kRowDim);
  plan_densify(rows, n, e->accum_norm, e->accum_cnt, dc, extent, seed, surv, children, counts, s);
  const int64_t nsurv = counts[0], nchild = counts[1], n2 = nsurv + nchild;
  require(n2 <= INT32_MAX, "densify: population overflow");
  const size_t nn = (size_t)std::max<int64_t>(n2, 1);
  float* gw2 = dmalloc<float>(nn * kGeoDim);
  float* gm2 = dmalloc<float>(nn * kGeoDim);
  float* gv2 = dmalloc<float>(nn * kGeoDim);
  uint8_t* gc2 = dmalloc<uint8_t>(nn);
  float* nw2 = nullptr;
  uint8_t* nc2 = nullptr;
  if (e->ng_host)
    GSS_CUDA(cudaHostAlloc((void**)&nw2, nn * kNgStride * 4, cudaHostAllocMapped));
  else
    nw2 = dmalloc<float>(nn * kNgStride);
  nc2 = dmalloc<uint8_t>(nn);
  if (n2 > 0) {
    densify_apply_kernel<<<(unsigned)ceil_div(n2, 256), 256, 0, s>>>(nsurv, nchild, surv, children, e->gw, e->gm,
                                                                    e->gv, e->gcnt, e->nw, e->ncnt, gw2, gm2, gv2,
                                                                    gc2, nw2, nc2);
    GSS_LAUNCHED();
  }
  GSS_CUDA(cudaStreamSynchronize(s));
  cudaFree(rows);
  cudaFree(surv);
  cudaFree(children);
  arena_release(&e->geo);
  arena_release(&e->ng);
  cudaFree(e->gw); cudaFree(e->gm); cudaFree(e->gv); cudaFree(e->gcnt);
  if (e->ng_host) cudaFreeHost(e->nw); else cudaFree(e->nw);
  cudaFree(e->ncnt);
  e->gw = gw2; e->gm = gm2; e->gv = gv2; e->gcnt = gc2;
  e->nw = nw2; e->nm = nw2 + kNgSeg; e->nv = nw2 + 2 * kNgSeg; e->ncnt = nc2;
  if (e->ng_host) {  // the concurrent host tier's row mask follows the population
    cudaFree(e->vis_mask);
    e->vis_mask = dmalloc<uint32_t>((nn + 31) / 32);
    GSS_CUDA(cudaMemset(e->vis_mask, 0, (nn + 31) / 32 * 4));
  }
  e->n = n2;
  e->geo.w = gw2; e->geo.m = gm2; e->geo.v = gv2; e->geo.counter = gc2; e->geo.n = n2;
  e->ng.w = e->nw; e->ng.m = e->nm; e->ng.v = e->nv; e->ng.counter = nc2; e->ng.n = n2;
  // n-sized per-iteration buffers and statistics
  for (int p = 0; p < 3; ++p) {
    cudaFree(e->ids[p]);
    e->ids[p] = dmalloc<int32_t>(nn);
  }
  cudaFree(e->cull_ws);
  e->cull_ws_bytes = cull_workspace_bytes(n2);
  e->cull_ws = dmalloc<char>(e->cull_ws_bytes);
  GSS_CUDA(cudaMemset(e->cull_ws, 0, e->cull_ws_bytes));
  cudaFree(e->accum_norm);
  cudaFree(e->accum_cnt);
  e->accum_norm = dmalloc<double>(nn);
  e->accum_cnt = dmalloc<int32_t>(nn);
  GSS_CUDA(cudaMemset(e->accum_norm, 0, nn * 8));
  GSS_CUDA(cudaMemset(e->accum_cnt, 0, nn * 4));
  // stage buffers hold rows of the old population: invalidate (engine.hpp:154-162)
  for (int b = 0; b < 2; ++b) {
    e->fwd_iter[b] = -1;
    e->g_iter[b] = -1;
    e->g_plan[b] = -1;
  }
  counts[5] = n2;
}

void engine_state(gss_engine* e, float* geo_w, float* ng_w, float* ng_m, float* ng_v, uint8_t* ng_counter,
                  int64_t* steps2) {
  require(e != nullptr, "engine: null");
  if (e->open_pending >= 0) drain(e);
  GSS_CUDA(cudaDeviceSynchronize());
  const size_t n = (size_t)e->n;
  if (geo_w) GSS_CUDA(cudaMemcpy(geo_w, e->gw, n * kGeoDim * 4, cudaMemcpyDefault));
  auto rows2d = [&](float* dst, const float* src) {  // strided tier rows -> packed n x 49
    if (dst && n) GSS_CUDA(cudaMemcpy2D(dst, kNgDim * 4, src, kNgStride * 4, kNgDim * 4, n, cudaMemcpyDefault));
  };
  rows2d(ng_w, e->nw);
  rows2d(ng_m, e->nm);
  rows2d(ng_v, e->nv);
  if (ng_counter) GSS_CUDA(cudaMemcpy(ng_counter, e->ncnt, n, cudaMemcpyDefault));
  if (steps2) {
    steps2[0] = e->geo.step;
    steps2[1] = e->ng.step;
  }
}

void engine_accum(gss_engine* e, double* norm, int32_t* cnt) {
  require(e != nullptr, "engine: null");
  GSS_CUDA(cudaDeviceSynchronize());
  if (norm) GSS_CUDA(cudaMemcpy(norm, e->accum_norm, (size_t)e->n * 8, cudaMemcpyDeviceToHost));
  if (cnt) GSS_CUDA(cudaMemcpy(cnt, e->accum_cnt, (size_t)e->n * 4, cudaMemcpyDeviceToHost));
}

void engine_stage_ms(gss_engine* e, double* out6) {
  require(e && out6, "engine: null");
  for (int i = 0; i < kStages; ++i) {
    out6[i] = e->stage_ms[i];
    e->stage_ms[i] = 0.0;
  }
}

int64_t engine_launches(gss_engine* e) { return e ? e->launches_last : 0; }

// Per-iteration timeline (engine.hpp:22-28 TimelineRow, 230-237): enabling records an epoch event;
// every stage interval collected afterwards (at each drain) becomes a row.
void engine_timeline_enable(gss_engine* e, bool on) {
  require(e != nullptr, "engine: null");
  if (e->open_pending >= 0) drain(e);
  GSS_CUDA(cudaDeviceSynchronize());
  collect_times(e);
  e->timeline.clear();
  e->timeline_on = on;
  if (on) {
    if (!e->epoch) GSS_CUDA(cudaEventCreate(&e->epoch));
    if (!e->touched_ring) e->touched_ring = dmalloc<int64_t>(kTouchedRing);
    GSS_CUDA(cudaMemset(e->touched_ring, 0, kTouchedRing * sizeof(int64_t)));
    e->touched_next = 0;
    GSS_CUDA(cudaEventRecord(e->epoch, e->sD));
  }
}
int64_t engine_timeline(gss_engine* e, gss_timeline_row* rows, int64_t cap) {
  require(e != nullptr, "engine: null");
  if (e->open_pending >= 0) drain(e);
  const int64_t n = (int64_t)e->timeline.size();
  if (rows) std::memcpy(rows, e->timeline.data(), (size_t)std::min(n, cap) * sizeof(gss_timeline_row));
  return n;
}
// Stage-delay injection (test instrumentation, see stage_delay_kernel): delays cycle per stage start.
void engine_stage_delays(gss_engine* e, const uint32_t* ns, int n) {
  require(e != nullptr && (n == 0 || ns), "engine: null");
  e->delays_ns.assign(ns, ns + n);
  e->delay_next = 0;
}

// Live timing of the engine's composite / sweep kernel launches (bench roofline of the dominant
// kernels): CUDA events on the render stream around each forward_kernel / backward_kernel.
void engine_kernel_timing(gss_engine* e, bool on) {
  require(e != nullptr, "engine: null");
  render_ctx_timing(e->rctx, on);
}
void engine_kernel_times(gss_engine* e, double* ms2, int64_t* n2, uint64_t* contribs, int nk) {
  require(e != nullptr, "engine: null");
  if (e->open_pending >= 0) drain(e);
  GSS_CUDA(cudaDeviceSynchronize());
  render_ctx_times(e->rctx, ms2, n2, contribs, nk);
}
int64_t engine_count(gss_engine* e) { return e ? e->n : 0; }

}  // namespace gssd
