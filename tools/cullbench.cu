// Standalone timing harness for cull.cu variants (dev only).
#include <atomic>
#include <string>
#include "../paper_2509_15645_b200/csrc/cull.cu"
namespace gssd {
void set_error(const std::string&) {}
void count_launch() {}
int64_t launches() { return 0; }
}
#include <algorithm>
#include <cstdio>
#include <vector>
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int64_t n; fread(&n, 8, 1, f);
  gss_camera cam; fread(&cam, sizeof cam, 1, f);
  std::vector<float> rows(n * 10); fread(rows.data(), 4, n * 10, f); fclose(f);
  float *geo; int32_t* ids; int64_t* cnt; void* ws;
  cudaMalloc(&geo, n * 40); cudaMemcpy(geo, rows.data(), n * 40, cudaMemcpyHostToDevice);
  cudaMalloc(&ids, n * 4); cudaMalloc(&cnt, 8);
  size_t wsb = gssd::cull_workspace_bytes(n); cudaMalloc(&ws, wsb); cudaMemset(ws, 0, wsb);
  gss_viewport vp{0.f, (float)cam.width, 0.f, (float)cam.height};
  cudaStream_t st; cudaStreamCreate(&st);
  for (int i = 0; i < 5; ++i) gssd::cull(geo, n, 10, &cam, &vp, 0.3f, nullptr, ids, cnt, ws, wsb, st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 50;
  cudaEventRecord(e0, st);
  for (int i = 0; i < reps; ++i) gssd::cull(geo, n, 10, &cam, &vp, 0.3f, nullptr, ids, cnt, ws, wsb, st);
  cudaEventRecord(e1, st); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  int64_t v; cudaMemcpy(&v, cnt, 8, cudaMemcpyDeviceToHost);
  printf("%s: %.2f us  visible %lld  %.0f GB/s\n", argv[2], ms * 1e3, (long long)v, (40.0 * n + 4.0 * v) / ms / 1e6);
#ifdef CULL_TRACE
  static unsigned long long tr[4096][6];
  cudaMemcpyFromSymbol(tr, gssd::g_cull_trace, sizeof(tr));
  int ctas = 0;
  while (ctas < 4096 && tr[ctas][0] != 0) ++ctas;
  unsigned long long t0 = ~0ull, qmax = 0, qsum = 0;
  for (int c = 0; c < ctas; ++c) { t0 = std::min(t0, tr[c][0]); qmax = std::max(qmax, tr[c][5]); qsum += tr[c][5]; }
  printf("ctas %d  queued rows: total %llu max per CTA %llu\n", ctas, qsum, qmax);
  for (int ph = 0; ph < 5; ++ph) {
    unsigned long long mn = ~0ull, mx = 0;
    double avg = 0;
    for (int c = 0; c < ctas; ++c) { mn = std::min(mn, tr[c][ph] - t0); mx = std::max(mx, tr[c][ph] - t0); avg += tr[c][ph] - t0; }
    printf("phase %d: min %.2f us  avg %.2f us  max %.2f us\n", ph, mn / 1e3, avg / ctas / 1e3, mx / 1e3);
  }
  // streaming-end time by CTA index (deciles) and the slowest CTAs with their queued-row counts
  for (int d = 0; d < 10; ++d) {
    double s1 = 0; int c0 = d * ctas / 10, c1 = (d + 1) * ctas / 10;
    for (int c = c0; c < c1; ++c) s1 += tr[c][1] - t0;
    printf("ctas %3d-%3d: stream end avg %.2f us\n", c0, c1 - 1, s1 / (c1 - c0) / 1e3);
  }
  for (int r = 0; r < 8; ++r) {
    int worst = 0;
    for (int c = 1; c < ctas; ++c) if (tr[c][1] > tr[worst][1]) worst = c;
    printf("slow cta %d: stream end %.2f us queued %llu start %.2f\n", worst, (tr[worst][1] - t0) / 1e3, tr[worst][5], (tr[worst][0]-t0)/1e3);
    tr[worst][1] = 0;
  }
#endif
  return 0;
}
