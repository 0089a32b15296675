// Streaming-read ceiling probes on 160 MB (dev only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_15645_b200/csrc/common.cuh"
namespace gssd { void set_error(const std::string&) {} void count_launch() {} int64_t launches() { return 0; } }
using namespace gssd;

template <int U>
__global__ void __launch_bounds__(256) rd_vec(const float4* __restrict__ p, int64_t n4, float* out) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n4; i += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (i + u * blockDim.x < n4) ? __ldcs(p + i + u * blockDim.x) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int STAGES, int BYTES>
__global__ void __launch_bounds__(256) rd_tma(const char* __restrict__ p, int64_t nbytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const int64_t nchunks = nbytes / BYTES;
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    for (int s = 0; s < STAGES; ++s) {
      int64_t c = blockIdx.x + (int64_t)s * G;
      if (c < nchunks) { mbar_expect_tx(&bar[s], BYTES); bulk_g2s(sm + s * BYTES, p + c * BYTES, BYTES, &bar[s]); }
    }
  }
  __syncthreads();
  float acc = 0.f;
  for (int j = 0;; ++j) {
    int64_t c = blockIdx.x + (int64_t)j * G;
    if (c >= nchunks) break;
    int s = j % STAGES;
    mbar_wait(&bar[s], (j / STAGES) & 1);
    const float* f = (const float*)(sm + s * BYTES);
    for (int i = threadIdx.x; i < BYTES / 4; i += 256) acc += f[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t c2 = blockIdx.x + (int64_t)(j + STAGES) * G;
      if (c2 < nchunks) { mbar_expect_tx(&bar[s], BYTES); bulk_g2s(sm + s * BYTES, p + c2 * BYTES, BYTES, &bar[s]); }
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

template <class F> void timeit(const char* name, F f, double bytes) {
  for (int i = 0; i < 5; ++i) f();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 50; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 50;
  printf("%-28s %8.2f us %7.0f GB/s\n", name, ms * 1e3, bytes / ms / 1e6);
}

int main() {
  const int64_t nbytes = 160000000LL;
  char* p; float* out; cudaMalloc(&p, nbytes + 4096); cudaMalloc(&out, 4); cudaMemset(p, 0, nbytes);
  char* q; cudaMalloc(&q, nbytes);
  const int64_t n4 = nbytes / 16;
  timeit("memcpy d2d (r+w)", [&] { cudaMemcpyAsync(q, p, nbytes, cudaMemcpyDeviceToDevice); }, 2.0 * nbytes);
  for (int g : {148 * 4, 148 * 8, 148 * 16}) {
    char nm[64]; snprintf(nm, 64, "vec U4 grid %d", g);
    timeit(nm, [&] { rd_vec<4><<<g, 256>>>((const float4*)p, n4, out); }, nbytes);
    snprintf(nm, 64, "vec U8 grid %d", g);
    timeit(nm, [&] { rd_vec<8><<<g, 256>>>((const float4*)p, n4, out); }, nbytes);
  }
  cudaFuncSetAttribute(rd_tma<4, 20480>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 20480);
  cudaFuncSetAttribute(rd_tma<8, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaFuncSetAttribute(rd_tma<2, 20480>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 20480);
  cudaFuncSetAttribute(rd_tma<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  timeit("tma 4x20K grid 296", [&] { rd_tma<4, 20480><<<296, 256, 4 * 20480>>>(p, nbytes, out); }, nbytes);
  timeit("tma 2x20K grid 592", [&] { rd_tma<2, 20480><<<592, 256, 2 * 20480>>>(p, nbytes, out); }, nbytes);
  timeit("tma 8x16K grid 148", [&] { rd_tma<8, 16384><<<148, 256, 8 * 16384>>>(p, nbytes, out); }, nbytes);
  timeit("tma 4x32K grid 148", [&] { rd_tma<4, 32768><<<148, 256, 4 * 32768>>>(p, nbytes, out); }, nbytes);
  timeit("tma 4x32K grid 296", [&] { rd_tma<4, 32768><<<296, 256, 4 * 32768>>>(p, nbytes, out); }, nbytes);
  // bigger buffer for reference: 1.6 GB
  return 0;
}
