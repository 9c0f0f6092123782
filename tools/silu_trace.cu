// Per-phase cycle stamps of the SiLU ISM kernel (CTA 0, thread 0, first 64 chunks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPIC_SILU_TRACE \
//        -o tools/silu_trace tools/silu_trace.cu
// Phases: 0 top, 1 records loaded, 2 F1 done (G1 issue), 3 previous chunk's F3 done,
// 4 G1 done, 5 F2a done, 6 per-particle done, 7 F2b done, 8 G2/G3 issued.
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2603_25832_b200/csrc/silu.cu"

namespace spic {
void count_launch() {}
__global__ void k_ism_reduce_cols(const double*, int, int64_t, double*) {}
}  // namespace spic

int main() {
  using namespace spic;
  const int64_t n = 1 << 20;
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
  return 0;
}
