// Per-phase cycle stamps of the SiLU ISM kernel (CTA 0, thread 0, first 64 chunks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPIC_SILU_TRACE \
//        -o tools/silu_trace tools/silu_trace.cu
// Phases: 0 top, 1 records loaded, 2 F1 done (G1 issue), 3 previous chunk's F3 done,
// 4 G1 done, 5 F2a done, 6 per-particle done, 7 F2b done, 8 G2/G3 issued.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include "../paper_2603_25832_b200/csrc/silu.cu"

namespace spic {
void count_launch() {}
__global__ void k_ism_reduce_cols(const double*, int, int64_t, double*) {}
}  // namespace spic

int main(int argc, char** argv) {
  using namespace spic;
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 20);
  const int P = (int)silu_params(kH);
  std::mt19937 g(1);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> params(P), rec(8 * n);
  for (auto& p : params) p = 0.1f * nd(g);
  for (int64_t i = 0; i < n; ++i) {
    rec[4 * i] = 31.4f * (float)i / n;
    for (int k = 1; k < 4; ++k) rec[4 * i + k] = nd(g);
    for (int k = 0; k < 3; ++k) rec[4 * n + 4 * i + k] = 0.f;
    rec[4 * n + 4 * i + 3] = 31.4f / n;
  }
  float *dp, *dr;
  double* part;
  cudaMalloc(&dp, P * 4);
  cudaMalloc(&dr, rec.size() * 4);
  cudaMalloc(&part, spic_silu_scratch_bytes(n));
  cudaMemcpy(dp, params.data(), P * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rec.data(), rec.size() * 4, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep)
    spic_silu_ism_partials(dp, kH, dr, dr + 4 * n, n, 1.f / 31.4f, part,
                           spic_silu_scratch_bytes(n), nullptr);
  cudaDeviceSynchronize();
  long long h[64 * 16];
  cudaMemcpyFromSymbol(h, g_silu_trace, sizeof(h));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));

  double sum[9] = {0};
  int cnt = 0;
  for (int it = 4; it < 63; ++it) {
    if (!h[(it + 1) * 16]) break;
    for (int k = 1; k <= 8; ++k) sum[k] += (double)(h[it * 16 + k] - h[it * 16 + k - 1]);
    sum[0] += (double)(h[(it + 1) * 16] - h[it * 16 + 8]);
    ++cnt;
  }
  const char* names[9] = {"loop-tail", "wait G3 + records", "F1", "F3(prev) under G1",
                          "G1 wait", "F2a", "per-particle", "F2b", "G2/G3 issue"};
  double tot = 0;
  for (int k = 0; k <= 8; ++k) tot += sum[k];
  for (int k = 0; k <= 8; ++k)
    printf("%-20s %8.0f cycles %5.1f%%\n", names[k], sum[k] / cnt, 100 * sum[k] / tot);
  printf("%-20s %8.0f cycles (%d chunks)\n", "chunk total", tot / cnt, cnt);
  // absolute offsets from the chunk's F1 hand-off (stamp 2): issuer and G2-arrival stamps
  double a9 = 0, a10 = 0, a11 = 0, a4 = 0, a12 = 0, a13 = 0, a7 = 0;
  for (int it = 4; it < 4 + cnt; ++it) {
    const double t2 = (double)h[it * 16 + 2];
    a10 += h[it * 16 + 10] - t2;   // issuer sees X ready
    a11 += h[it * 16 + 11] - t2;   // G1 issued
    a9 += h[(it + 1) * 16 + 9] - (double)h[(it + 1) * 16 + 2];  // next chunk: F3 got G2(prev)
    a4 += h[it * 16 + 4] - t2;     // G1 complete seen by compute
    a7 += h[it * 16 + 7] - t2;     // F2b done
    a12 += h[it * 16 + 12] - t2;   // issuer sees Y ready
    a13 += h[it * 16 + 13] - t2;   // G3 + G2 issued
  }
  double a14 = 0;
  for (int it = 4; it < 4 + cnt; ++it) a14 += h[it * 16 + 14] - (double)h[it * 16 + 12];
  if (h[4 * 16 + 14]) printf("G3 complete %.0f cycles after the issuer saw Y ready\n", a14 / cnt);
  printf("kernel (CTA 0): prologue %lld, chunk loop %lld, epilogue %lld cycles\n",
         h[63 * 16 + 1] - h[63 * 16 + 0], h[63 * 16 + 2] - h[63 * 16 + 1],
         h[63 * 16 + 3] - h[63 * 16 + 2]);
  printf("epilogue: G3 wait+sync %lld, tangent/dW2 rows %lld, combine %lld, dW1 tangent %lld, "
         "final rows %lld\n", h[63 * 16 + 4] - h[63 * 16 + 2], h[63 * 16 + 5] - h[63 * 16 + 4],
         h[63 * 16 + 6] - h[63 * 16 + 5], h[63 * 16 + 7] - h[63 * 16 + 6],
         h[63 * 16 + 3] - h[63 * 16 + 7]);
  if (h[63 * 16 + 12])
    printf("epilogue dW2 block, first half: TMEM loads %lld, flushed sums + W2 row %lld, 16 columns %lld, "
           "row stores %lld\n", h[63 * 16 + 9] - h[63 * 16 + 8], h[63 * 16 + 10] - h[63 * 16 + 9],
           h[63 * 16 + 11] - h[63 * 16 + 10], h[63 * 16 + 12] - h[63 * 16 + 11]);
  printf("from F1 hand-off: issuer X-ready %+.0f, G1 issued %+.0f, G1 done %+.0f, F2b done %+.0f,\n"
         "  issuer Y-ready %+.0f, G3+G2 issued %+.0f; next chunk's F3 got G2 %+.0f after its F1 hand-off\n",
         a10 / cnt, a11 / cnt, a4 / cnt, a7 / cnt, a12 / cnt, a13 / cnt, a9 / cnt);
  return 0;
}
