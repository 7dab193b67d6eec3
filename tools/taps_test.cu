// taps_test.cu — standalone check of gemm_tc.cu's tap modes against a CPU product (tool).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1602_08191_b200/csrc/gemm_tc.cu"
#include "../paper_1602_08191_b200/csrc/capi.cu"

int main(int argc, char** argv) {
  using namespace dsb;
  const uint32_t M = argc > 1 ? atoi(argv[1]) : 128, N = argc > 2 ? atoi(argv[2]) : 192, K = argc > 3 ? atoi(argv[3]) : 50;
  const int T = argc > 4 ? atoi(argv[4]) : 9, splits = argc > 5 ? atoi(argv[5]) : 1;
  const uint64_t ld = (K + 3) / 4 * 4;
  std::vector<float> A(M * ld), B(N * ld), D(M * N * (T > 0 ? T : 1), -7.f);
  srand(1);
  for (auto& v : A) v = (rand() % 2001 - 1000) / 1000.f;
  for (auto& v : B) v = (rand() % 2001 - 1000) / 1000.f;
  float *dA, *dB, *dD, *part;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMalloc(&part, 64ull << 20);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice);
  if (T == 0) {  // plain GEMM, D [M x N]
    GemmEpilogue ep0;
    ep0.D = dD;
    ep0.ldd = N;
    int rc0 = launch_gemm_tf32(dA, ld, dB, ld, M, N, K, ep0, 1, nullptr, 0);
    cudaError_t e0 = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, 4ull * M * N, cudaMemcpyDeviceToHost);
    double me = 0;
    if (1.0 * M * N * K < 1e9)
    for (uint32_t m = 0; m < M; ++m)
      for (uint32_t n = 0; n < N; ++n) {
        double r = 0;
        for (uint32_t k = 0; k < K; ++k) r += A[m * ld + k] * B[n * ld + k];
        me = fmax(me, fabs(r - D[m * N + n]));
      }
    printf("plain M %u N %u K %u (rc %d, %s): max err %.3e\n", M, N, K, rc0, cudaGetErrorString(e0), me);
    cudaEvent_t e1, e2;
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    for (int it = 0; it < 3; ++it) launch_gemm_tf32(dA, ld, dB, ld, M, N, K, ep0, 1, nullptr, 0);
    cudaEventRecord(e1);
    for (int it = 0; it < 20; ++it) launch_gemm_tf32(dA, ld, dB, ld, M, N, K, ep0, 1, nullptr, 0);
    cudaEventRecord(e2);
    cudaEventSynchronize(e2);
    float ms = 0;
    cudaEventElapsedTime(&ms, e1, e2);
    printf("  %.1f TFLOP/s (bn %u)\n", 2.0 * M * N * K * 20 / (ms / 1e3) / 1e12, gemm_pick_bn(N));
    return 0;
  }
  if (getenv("ACC_TAPS")) {  // accumulate mode: D[m][n] = sum_t sum_k A[m + sh_t][k] B[n][t*K + k]
    const int SH[9] = {-17, -16, -15, -1, 0, 1, 15, 16, 17};
    std::vector<float> Bt(static_cast<size_t>(N) * T * K), Dt(static_cast<size_t>(M) * N, -7.f);
    for (auto& v : Bt) v = (rand() % 2001 - 1000) / 1000.f;
    float *dBt, *dDt;
    cudaMalloc(&dBt, Bt.size() * 4);
    cudaMalloc(&dDt, Dt.size() * 4);
    cudaMemcpy(dBt, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
    GemmTaps ta;
    ta.n = T;
    ta.kt = K;
    for (int t = 0; t < T; ++t) ta.a_row[t] = SH[t % 9], ta.a_col[t] = 0, ta.b_row[t] = 0, ta.b_col[t] = t * K;
    GemmEpilogue e1;
    e1.D = dDt;
    e1.ldd = N;
    GemmOperand a1{dA, M, K, ld}, b1{dBt, N, static_cast<uint64_t>(T) * K, static_cast<uint64_t>(T) * K};
    int rc1 = launch_gemm(a1, b1, M, N, 0, &ta, e1, 1, nullptr, 0);
    cudaError_t ee = cudaDeviceSynchronize();
    cudaMemcpy(Dt.data(), dDt, Dt.size() * 4, cudaMemcpyDeviceToHost);
    double me = 0;
    for (uint32_t m = 0; m < M; ++m)
      for (uint32_t n = 0; n < N; ++n) {
        double r = 0;
        for (int t = 0; t < T; ++t) {
          const int mm = static_cast<int>(m) + SH[t % 9];
          if (mm < 0 || mm >= static_cast<int>(M)) continue;
          for (uint32_t k = 0; k < K; ++k) r += A[mm * ld + k] * Bt[(static_cast<size_t>(n) * T + t) * K + k];
        }
        me = fmax(me, fabs(r - Dt[m * N + n]));
      }
    printf("acc taps %d M %u N %u K %u (rc %d, %s, halo %s): max err %.3e\n", T, M, N, K, rc1, cudaGetErrorString(ee),
           getenv("DS_GEMM_HALO") ? getenv("DS_GEMM_HALO") : "0", me);
    return 0;
  }
  GemmTaps tp;
  tp.n = T;
  tp.per_z = 1;
  tp.d_col_step = N;
  for (int t = 0; t < T; ++t) tp.a_row[t] = tp.a_col[t] = tp.b_row[t] = 0, tp.b_col[t] = 4 * (t - T / 2);
  GemmEpilogue ep;
  ep.D = dD;
  ep.ldd = N * T;
  GemmOperand a{dA, M, K, ld}, b{dB, N, K, ld};
  int rc = launch_gemm(a, b, M, N, K, &tp, ep, splits, part, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("rc %d (%s) sync %s\n", rc, last_error().c_str(), cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int t = 0; t < T; ++t)
    for (uint32_t m = 0; m < M; ++m)
      for (uint32_t n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < static_cast<int>(K); ++k) {
          const int kb = k + 4 * (t - T / 2);
          if (kb >= 0 && kb < static_cast<int>(K)) r += A[m * ld + k] * B[n * ld + kb];
        }
        maxerr = fmax(maxerr, fabs(r - D[m * N * T + t * N + n]));
      }
  printf("per_z taps %d M %u N %u K %u splits %d: max err %.3e\n", T, M, N, K, splits, maxerr);
  return 0;
}
