// Empirical check (dev only): Markstein division with a correctly rounded reciprocal,
//   q0 = a*y, r = fma(-b, q0, a), q = fma(r, y, q0), y = RN(1/b)
// equals IEEE a/b (div.rn) for random a, b in the guarded range. Prints the mismatch count.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hash(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}
__global__ void k(uint64_t seed, int64_t n, unsigned long long* bad, int mode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t ha = hash(seed * 0x9E3779B97F4A7C15ull + 2 * i), hb = hash(seed * 0x9E3779B97F4A7C15ull + 2 * i + 1);
    float a, b;
    if (mode == 0) {  // uniform over bit patterns in [2^-60, 2^60]
      a = __uint_as_float(((ha % (120u << 23)) + ((127u - 60u) << 23)));
      b = __uint_as_float(((hb % (120u << 23)) + ((127u - 60u) << 23)));
    } else {  // b with all-ones-ish mantissas near powers of two (hard cases)
      a = __uint_as_float(((ha % (40u << 23)) + ((127u - 20u) << 23)));
      b = __uint_as_float((((hb % 40u) + 107u) << 23) | (0x7fffffu - (hb >> 28)));
    }
    const float y = __frcp_rn(b);
    const float q0 = __fmul_rn(a, y);
    const float r = __fmaf_rn(-b, q0, a);
    const float q = __fmaf_rn(r, y, q0);
    const float ref = __fdiv_rn(a, b);
    if (__float_as_uint(q) != __float_as_uint(ref)) atomicAdd(bad, 1ull);
  }
}
int main() {
  unsigned long long* bad; cudaMalloc(&bad, 8);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(bad, 0, 8);
    for (int s = 0; s < 20; ++s) k<<<148 * 16, 256>>>(s + 1, 1ll << 28, bad, mode);
    unsigned long long h; cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %llu mismatches in %lld pairs\n", mode, h, 20ll << 28);
  }
  return 0;
}
