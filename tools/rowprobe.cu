// Access-pattern ceiling of the non-geometric tier's row walks (dev only): the deferred walk and the
// forwarding gather read (and the walk writes back) the 624-B w/m/v span of listed rows of a
// 40M x 160-float row-interleaved arena, the list ascending with density f. This probe moves the
// same bytes with no arithmetic — warps walk 32 listed rows x 39 float4 units, U units per lane in
// flight — so its GB/s is the ceiling the optimizer kernels can reach for that access pattern.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rowprobe tools/rowprobe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int kStride = 160, kUnits = 39;  // floats per row, float4 units of the w..v span

template <int U, bool WRITE>
__global__ void __launch_bounds__(256) walk(float* __restrict__ a, const int32_t* __restrict__ rows, int64_t T,
                                            float* out) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  const int64_t wstride = (int64_t)gridDim.x * 8 * 32;
  for (int64_t t0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32; t0 < T; t0 += wstride) {
    const int64_t my = t0 + lane < T ? (int64_t)rows[t0 + lane] * kStride : -1;
    // flattened (row, unit) space of the 32 rows: 32 * 39 units, lane l takes l, l + 32, ...
    for (int i0 = lane; i0 < 32 * kUnits; i0 += 32 * U) {
      float4 v[U];
      int64_t o[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + 32 * u;
        const int r = i / kUnits, q = i - r * kUnits;
        const int64_t base = __shfl_sync(0xffffffffu, my, r < 32 ? r : 31);
        o[u] = (i < 32 * kUnits && base >= 0) ? base + 4 * q : -1;
        v[u] = o[u] >= 0 ? *reinterpret_cast<const float4*>(a + o[u]) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (WRITE) {
          if (o[u] >= 0) {
            float4 w = v[u];
            w.x *= 1.0001f;
            *reinterpret_cast<float4*>(a + o[u]) = w;
          }
        } else {
          acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
      }
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int U, bool WRITE>
double run(float* a, const int32_t* rows, int64_t T, float* out, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  walk<U, WRITE><<<blocks, 256>>>(a, rows, T, out);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) walk<U, WRITE><<<blocks, 256>>>(a, rows, T, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)T * kUnits * 16 * (WRITE ? 2 : 1);
  return bytes / (ms / reps / 1e3) / 1e9;
}

int main() {
  const int64_t n = 40000000;
  float* a;
  float* out;
  if (cudaMalloc(&a, (size_t)n * kStride * 4) != cudaSuccess) return 1;
  cudaMemset(a, 0, (size_t)n * kStride * 4);
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int32_t* rows;
  cudaMalloc(&rows, (size_t)n * 4);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (double f : {0.129, 0.5, 1.0}) {
    std::vector<int32_t> h;
    h.reserve((size_t)(n * f) + 16);
    for (int64_t i = 0; i < n; ++i) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      if ((double)(s >> 11) * (1.0 / 9007199254740992.0) < f) h.push_back((int32_t)i);
    }
    cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const int64_t T = (int64_t)h.size();
    for (int bpsm : {4, 8}) {
      const int blocks = sms * bpsm;
      printf("f %.3f rows %lld blocks/SM %d | read GB/s U1 %.0f U2 %.0f U4 %.0f | read+write GB/s U1 %.0f U2 %.0f U4 %.0f\n",
             f, (long long)T, bpsm, run<1, false>(a, rows, T, out, blocks), run<2, false>(a, rows, T, out, blocks),
             run<4, false>(a, rows, T, out, blocks), run<1, true>(a, rows, T, out, blocks),
             run<2, true>(a, rows, T, out, blocks), run<4, true>(a, rows, T, out, blocks));
    }
  }
  const cudaError_t err = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
