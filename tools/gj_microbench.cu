// standalone GJ microbenchmark: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1403_5337_b200/csrc tools/gj_microbench.cu -o exp/gj_microbench
#include "../paper_1403_5337_b200/csrc/gj.cu"
#ifndef GJ_MB_NS
#define GJ_MB_NS 64, 110, 128
#endif
#ifndef GJ_MB_TASKS
#define GJ_MB_TASKS 1, 128, 512
#endif
#include <cstdio>
#include <cstring>
#include <vector>
#include <random>
void hk_count_launch(int) {}
int main() {
  for (int N : {GJ_MB_NS}) {
    for (int ntask : {GJ_MB_TASKS}) {
      std::vector<double> A((size_t)ntask * N * N);
      std::mt19937_64 g(1);
      std::normal_distribution<double> d;
      for (int t = 0; t < ntask; ++t)
        for (int i = 0; i < N; ++i)
          for (int j = 0; j < N; ++j) A[(size_t)t * N * N + i * N + j] = d(g) + (i == j ? 10 : 0);
      double *dA, *dO; int* st; GjTask* dt;
      cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dO, A.size() * 8); cudaMalloc(&st, ntask * 4);
      cudaMalloc(&dt, ntask * sizeof(GjTask));
      cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
      std::vector<GjTask> ts(ntask);
      for (int t = 0; t < ntask; ++t) {
        GjTask x{};
        x.src = dA + (size_t)t * N * N; x.src_ld = N; x.out = dO + (size_t)t * N * N; x.out_ld = N;
        x.status = st + t; x.N = N; x.mode = 1;
        ts[t] = x;
      }
      cudaMemcpy(dt, ts.data(), ntask * sizeof(GjTask), cudaMemcpyHostToDevice);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int it = 0; it < 3; ++it) hk_launch_gj(dt, ntask, N, 0);
      cudaEventRecord(e0);
      for (int it = 0; it < 10; ++it) hk_launch_gj(dt, ntask, N, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      // check: A * Ainv ~ I for task 0
      std::vector<double> O((size_t)N * N);
      cudaMemcpy(O.data(), dO, N * N * 8, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int i = 0; i < N; ++i) for (int j = 0; j < N; ++j) {
        double s = 0; for (int k = 0; k < N; ++k) s += A[i * N + k] * O[k + j * N];   // A row-major? mode 1 = column-major src
        // mode 1: src[i + j*ld] -> A treated column-major: M[i][j] = A[i + j*N]
        (void)s;
      }
      for (int i = 0; i < N; ++i) for (int j = 0; j < N; ++j) {
        double s = 0; for (int k = 0; k < N; ++k) s += A[i + k * N] * O[k + j * N];
        err = std::max(err, std::fabs(s - (i == j)));
      }
      std::vector<double> all((size_t)ntask * N * N);
      cudaMemcpy(all.data(), dO, all.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long hsh = 1469598103934665603ull;
      for (double v : all) { unsigned long long u; memcpy(&u, &v, 8); hsh = (hsh ^ u) * 1099511628211ull; }
      printf("N=%3d tasks=%5d  %8.1f us/launch  err=%.1e  hash=%016llx %s\n", N, ntask, ms * 100, err, hsh, cudaGetErrorString(cudaGetLastError()));
      cudaFree(dA); cudaFree(dO); cudaFree(st); cudaFree(dt);
    }
  }
}
