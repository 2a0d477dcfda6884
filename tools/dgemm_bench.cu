// Times K2's two fp64 GEMM shapes (batched over 24 heads) on our DMMA kernel
// (gemm_f64.cu, compiled in) against cuBLAS DGEMM, and checks agreement.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/dgemm_bench.cu -o tools/dgemm_bench -lcublas
#include "../paper_2511_19835_b200/csrc/gemm_f64.cu"

#include <cublas_v2.h>
#include <cstdio>
#include <vector>
#include <cmath>

int main() {
  const int H = 24;
  struct Case { const char* name; int64_t M, N, K; bool nt; } cases[] = {
      {"scores NT 928x1184x128", 928, 1184, 128, true},
      {"comp   NN 928x128x930 ", 928, 128, 930, false}};
  cublasHandle_t hb;
  cublasCreate(&hb);
  for (auto& c : cases) {
    const int64_t sa = c.M * c.K, sb = c.N * c.K, sc = c.M * c.N;
    std::vector<double> hA(H * sa), hB(H * sb);
    for (auto& x : hA) x = (double)rand() / RAND_MAX - 0.5;
    for (auto& x : hB) x = (double)rand() / RAND_MAX - 0.5;
    double *A, *B, *C1, *C2;
    cudaMalloc(&A, H * sa * 8); cudaMalloc(&B, H * sb * 8); cudaMalloc(&C1, H * sc * 8); cudaMalloc(&C2, H * sc * 8);
    cudaMemcpy(A, hA.data(), H * sa * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB.data(), H * sb * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int cfg = 0;
    auto ours = [&]() {
      rsa::GemmArgs ga{c.M, c.N, c.K, A, c.K, sa, B, c.nt ? c.K : c.N, sb, C1, c.N, sc};
      rsa::launch_dgemm_cfg(ga, H, c.nt, 0, cfg);
    };
    const double one = 1.0, zero = 0.0;
    auto theirs = [&]() {
      if (c.nt)
        cublasDgemmStridedBatched(hb, CUBLAS_OP_T, CUBLAS_OP_N, c.N, c.M, c.K, &one, B, c.K, sb, A, c.K, sa, &zero,
                                  C2, c.N, sc, H);
      else
        cublasDgemmStridedBatched(hb, CUBLAS_OP_N, CUBLAS_OP_N, c.N, c.M, c.K, &one, B, c.N, sb, A, c.K, sa, &zero,
                                  C2, c.N, sc, H);
    };
    for (cfg = 1; cfg <= 9; ++cfg) {
    if (cfg == 9) cfg = 0;
    for (int w = 0; w < 3; ++w) { ours(); theirs(); }
    float t_o = 0, t_c = 0;
    const int R = 20;
    cudaEventRecord(e0); for (int r = 0; r < R; ++r) ours(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t_o, e0, e1);
    cudaEventRecord(e0); for (int r = 0; r < R; ++r) theirs(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t_c, e0, e1);
    std::vector<double> h1(H * sc), h2(H * sc);
    cudaMemcpy(h1.data(), C1, H * sc * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), C2, H * sc * 8, cudaMemcpyDeviceToHost);
    double md = 0;
    for (size_t i = 0; i < h1.size(); ++i) md = std::fmax(md, std::fabs(h1[i] - h2[i]));
    const double fl = 2.0 * H * c.M * c.N * c.K;
    printf("cfg %d %s  ours %.3f ms (%.1f TF/s)  cublas %.3f ms (%.1f TF/s)  max|diff| %.2e  err=%s\n", cfg, c.name, t_o / R,
           fl / (t_o / R * 1e-3) / 1e12, t_c / R, fl / (t_c / R * 1e-3) / 1e12, md,
           cudaGetErrorString(cudaGetLastError()));
    if (cfg == 0) break;
    }
    cudaFree(A); cudaFree(B); cudaFree(C1); cudaFree(C2);
  }
  return 0;
}
