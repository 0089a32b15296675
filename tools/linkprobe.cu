// Host-link ceiling probes (dev only): pinned cudaMemcpyAsync H2D / D2H / both directions at once,
// and SM-driven zero-copy access to mapped pinned memory (scattered 640-byte rows, the host-tier
// layout): gather (host -> device), scatter (device -> host), and both in one kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/linkprobe tools/linkprobe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <chrono>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int kRowF4 = 40;  // 640 B

__global__ void gather_rows(const float4* __restrict__ host, const int32_t* ids, int64_t nids, float4* out) {
  const int64_t total = nids * kRowF4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / kRowF4;
    const int u = (int)(i - k * kRowF4);
    out[i] = host[(int64_t)ids[k] * kRowF4 + u];
  }
}
__global__ void scatter_rows(float4* host, const int32_t* ids, int64_t nids, const float4* __restrict__ in) {
  const int64_t total = nids * kRowF4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / kRowF4;
    const int u = (int)(i - k * kRowF4);
    host[(int64_t)ids[k] * kRowF4 + u] = in[i];
  }
}
// read row, modify, write back in place (the fused lazy-update access pattern)
__global__ void rmw_rows(float4* host, const int32_t* ids, int64_t nids) {
  const int64_t total = nids * kRowF4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / kRowF4;
    const int u = (int)(i - k * kRowF4);
    float4 v = host[(int64_t)ids[k] * kRowF4 + u];
    v.x += 1.0f;
    host[(int64_t)ids[k] * kRowF4 + u] = v;
  }
}

// Few-CTA zero-copy row movers: each thread keeps 8 independent 16-byte transfers in flight, so a
// small grid (leaving the other SMs to compute) can still saturate the link.
template <bool GATHER>
__global__ void __launch_bounds__(256) move_rows_ilp(float4* host, const int32_t* ids, int64_t nids, float4* dev) {
  const int64_t total = nids * kRowF4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < total; base += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = base + u * stride;
      if (i < total) {
        const int64_t k = i / kRowF4;
        const int c = (int)(i - k * kRowF4);
        v[u] = GATHER ? host[(int64_t)ids[k] * kRowF4 + c] : dev[i];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = base + u * stride;
      if (i < total) {
        const int64_t k = i / kRowF4;
        const int c = (int)(i - k * kRowF4);
        if (GATHER) dev[i] = v[u]; else host[(int64_t)ids[k] * kRowF4 + c] = v[u];
      }
    }
  }
}

int main(int argc, char** argv) {
  const size_t big = (size_t)1 << 30;  // 1 GiB
  char *h1, *h2, *d1, *d2;
  CK(cudaHostAlloc((void**)&h1, big, cudaHostAllocDefault));
  CK(cudaHostAlloc((void**)&h2, big, cudaHostAllocDefault));
  CK(cudaMalloc(&d1, big));
  CK(cudaMalloc(&d2, big));
  memset(h1, 1, big);
  memset(h2, 2, big);
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto timeit = [&](auto fn, int reps) {
    fn();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, 0));
    for (int r = 0; r < reps; ++r) fn();
    CK(cudaEventRecord(b, 0));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
  };
  for (size_t chunk : {(size_t)32 << 20, big}) {
    const int nc = (int)(big / chunk);
    float ms = timeit([&] { for (int c = 0; c < nc; ++c) CK(cudaMemcpyAsync(d1 + c * chunk, h1 + c * chunk, chunk, cudaMemcpyHostToDevice, 0)); }, 5);
    printf("{\"probe\":\"memcpy_h2d\",\"chunk_mb\":%zu,\"gbs\":%.2f}\n", chunk >> 20, big / ms / 1e6);
    ms = timeit([&] { for (int c = 0; c < nc; ++c) CK(cudaMemcpyAsync(h2 + c * chunk, d2 + c * chunk, chunk, cudaMemcpyDeviceToHost, 0)); }, 5);
    printf("{\"probe\":\"memcpy_d2h\",\"chunk_mb\":%zu,\"gbs\":%.2f}\n", chunk >> 20, big / ms / 1e6);
  }
  {  // both directions concurrently on two streams
    cudaEvent_t j;
    CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
    float ms = timeit([&] {
      CK(cudaEventRecord(j, 0));
      CK(cudaStreamWaitEvent(s1, j, 0));
      CK(cudaStreamWaitEvent(s2, j, 0));
      CK(cudaMemcpyAsync(d1, h1, big, cudaMemcpyHostToDevice, s1));
      CK(cudaMemcpyAsync(h2, d2, big, cudaMemcpyDeviceToHost, s2));
      CK(cudaEventRecord(j, s1));
      CK(cudaStreamWaitEvent(0, j, 0));
      CK(cudaEventRecord(j, s2));
      CK(cudaStreamWaitEvent(0, j, 0));
    }, 5);
    printf("{\"probe\":\"memcpy_bidir\",\"gbs_each_way\":%.2f,\"gbs_total\":%.2f}\n", big / ms / 1e6, 2 * big / ms / 1e6);
  }
  // zero-copy on a mapped 6.4 GB arena of 10M rows x 640 B, 14% of the rows (random, ascending)
  const int64_t nrows = 10'000'000;
  float4* harena;
  CK(cudaHostAlloc((void**)&harena, (size_t)nrows * 640, cudaHostAllocMapped));
  memset(harena, 0, (size_t)nrows * 640);
  float4* darena_view;
  CK(cudaHostGetDevicePointer((void**)&darena_view, harena, 0));
  std::vector<int32_t> ids;
  std::mt19937 rng(1);
  for (int64_t i = 0; i < nrows; ++i) if ((rng() % 100) < 14) ids.push_back((int32_t)i);
  int32_t* dids;
  CK(cudaMalloc(&dids, ids.size() * 4));
  CK(cudaMemcpy(dids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice));
  float4* dout;
  CK(cudaMalloc(&dout, ids.size() * 640));
  const int64_t nids = (int64_t)ids.size();
  const double bytes = (double)nids * 640;
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    float ms = timeit([&] { gather_rows<<<blocks, 512>>>(darena_view, dids, nids, dout); }, 3);
    printf("{\"probe\":\"zc_gather\",\"blocks\":%d,\"rows\":%lld,\"gbs\":%.2f}\n", blocks, (long long)nids, bytes / ms / 1e6);
    ms = timeit([&] { scatter_rows<<<blocks, 512>>>(darena_view, dids, nids, dout); }, 3);
    printf("{\"probe\":\"zc_scatter\",\"blocks\":%d,\"gbs\":%.2f}\n", blocks, bytes / ms / 1e6);
    ms = timeit([&] { rmw_rows<<<blocks, 512>>>(darena_view, dids, nids); }, 3);
    printf("{\"probe\":\"zc_rmw\",\"blocks\":%d,\"gbs_each_way\":%.2f}\n", blocks, bytes / ms / 1e6);
  }
  {  // gather and scatter on two streams at once (different row sets)
    float ms = timeit([&] {
      gather_rows<<<148 * 8, 512, 0, s1>>>(darena_view, dids, nids / 2, dout);
      scatter_rows<<<148 * 8, 512, 0, s2>>>(darena_view, dids + nids / 2, nids - nids / 2, dout);
      CK(cudaStreamSynchronize(s1));
      CK(cudaStreamSynchronize(s2));
    }, 3);
    printf("{\"probe\":\"zc_gather_scatter_concurrent\",\"gbs_total\":%.2f}\n", bytes / ms / 1e6);
  }
  for (int blocks : {8, 16, 32, 64, 128}) {
    float ms = timeit([&] { move_rows_ilp<true><<<blocks, 256>>>(darena_view, dids, nids, dout); }, 3);
    printf("{\"probe\":\"zc_gather_ilp\",\"blocks\":%d,\"gbs\":%.2f}\n", blocks, bytes / ms / 1e6);
    ms = timeit([&] { move_rows_ilp<false><<<blocks, 256>>>(darena_view, dids, nids, dout); }, 3);
    printf("{\"probe\":\"zc_scatter_ilp\",\"blocks\":%d,\"gbs\":%.2f}\n", blocks, bytes / ms / 1e6);
  }
  {  // ILP gather (32 CTAs) + scatter (32 CTAs) concurrently, and gather (SM) + a contiguous CE D2H
    float ms = timeit([&] {
      move_rows_ilp<true><<<32, 256, 0, s1>>>(darena_view, dids, nids / 2, dout);
      move_rows_ilp<false><<<32, 256, 0, s2>>>(darena_view, dids + nids / 2, nids - nids / 2, dout);
      CK(cudaStreamSynchronize(s1));
      CK(cudaStreamSynchronize(s2));
    }, 3);
    printf("{\"probe\":\"zc_ilp_gather_scatter_concurrent\",\"gbs_total\":%.2f}\n", bytes / ms / 1e6);
    const size_t half = (size_t)(nids / 2) * 640;
    ms = timeit([&] {
      move_rows_ilp<true><<<32, 256, 0, s1>>>(darena_view, dids, nids / 2, dout);
      CK(cudaMemcpyAsync(h2, d2, half, cudaMemcpyDeviceToHost, s2));
      CK(cudaStreamSynchronize(s1));
      CK(cudaStreamSynchronize(s2));
    }, 3);
    printf("{\"probe\":\"zc_gather_plus_ce_d2h\",\"gbs_total\":%.2f}\n", 2 * half / ms / 1e6);
  }
  // (a copy-engine per-row gather probe was measured once at 0.82 GB/s, profiles/r02_linkprobe.txt;
  //  the batched-copy call it used is closed on this pool and the probe was removed)
  return 0;
}
