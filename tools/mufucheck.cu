// Exactness facts the backward sweep's neutral idle lanes rely on (GSS_BWD_NEUTRAL): MUFU.RCP of
// 1.0 is exactly 1.0 and MUFU.EX2 of -inf is exactly +0. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cmath>
#include <cstring>
__global__ void k(float* out) {
  float a = 1.0f, b = -INFINITY, r, e;
  asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-0.72134752f * (-b)));
  out[0] = r;
  out[1] = e;
  float one_minus_zero = 1.0f - 0.0f * 0.5f;
  asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(one_minus_zero));
  out[2] = r;
}
int main() {
  float* d; float h[3];
  cudaMalloc(&d, 12);
  k<<<1, 1>>>(d);
  cudaMemcpy(h, d, 12, cudaMemcpyDeviceToHost);
  unsigned u0, u1, u2; memcpy(&u0, &h[0], 4); memcpy(&u1, &h[1], 4); memcpy(&u2, &h[2], 4);
  printf("{\"rcp_1\": \"%08x\", \"ex2_neg_inf\": \"%08x\", \"rcp_1b\": \"%08x\", \"ok\": %s}\n", u0, u1, u2,
         (u0 == 0x3f800000u && u1 == 0u && u2 == 0x3f800000u) ? "true" : "false");
  return (u0 == 0x3f800000u && u1 == 0u && u2 == 0x3f800000u) ? 0 : 1;
}
