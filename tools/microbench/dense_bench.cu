// Timing of the cuSOLVER/cuBLAS pieces of the ChFSI loop at the BASELINE
// panel widths: zheevd vs zheevj (random and nearly-diagonal Hermitian),
// Householder QR (geqrf+ungqr) vs one Cholesky-QR pass (herk+potrf+trsm).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    auto e = (x);                                                           \
    if ((int)e != 0) {                                                      \
      printf("error %d at %s:%d\n", (int)e, __FILE__, __LINE__);            \
      exit(1);                                                              \
    }                                                                       \
  } while (0)

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  cusolverDnHandle_t sol;
  cublasHandle_t blas;
  CK(cusolverDnCreate(&sol));
  CK(cublasCreate(&blas));
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  int* info;
  cudaMalloc(&info, sizeof(int));
  for (int n : {32, 64, 100, 160, 300, 600, 1400, 3400}) {
    for (int kind = 0; kind < 2; ++kind) {
      std::vector<cuDoubleComplex> h((size_t)n * n);
      for (int j = 0; j < n; ++j)
        for (int i = 0; i <= j; ++i) {
          double re = nd(rng), im = i == j ? 0 : nd(rng);
          double s = kind ? 1e-6 : 1.0;
          re *= s;
          im *= s;
          if (i == j && kind) re += j;
          h[(size_t)j * n + i] = make_cuDoubleComplex(re, im);
          h[(size_t)i * n + j] = make_cuDoubleComplex(re, -im);
        }
      cuDoubleComplex *d, *w0;
      double* ev;
      cudaMalloc(&d, sizeof(cuDoubleComplex) * n * n);
      cudaMalloc(&w0, sizeof(cuDoubleComplex) * n * n);
      cudaMalloc(&ev, sizeof(double) * n);
      cudaMemcpy(w0, h.data(), sizeof(cuDoubleComplex) * n * n, cudaMemcpyHostToDevice);
      int lw = 0;
      CK(cusolverDnZheevd_bufferSize(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d, n, ev, &lw));
      cuDoubleComplex* work;
      cudaMalloc(&work, sizeof(cuDoubleComplex) * lw);
      float t_evd = time_ms([&] {
        cudaMemcpyAsync(d, w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice);
        cusolverDnZheevd(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d, n, ev, work, lw, info);
      });
      syevjInfo_t params;
      CK(cusolverDnCreateSyevjInfo(&params));
      cusolverDnXsyevjSetTolerance(params, 1e-15);
      cusolverDnXsyevjSetMaxSweeps(params, 20);
      int lwj = 0;
      CK(cusolverDnZheevj_bufferSize(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d, n, ev, &lwj, params));
      cuDoubleComplex* workj;
      cudaMalloc(&workj, sizeof(cuDoubleComplex) * lwj);
      float t_evj = time_ms([&] {
        cudaMemcpyAsync(d, w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice);
        cusolverDnZheevj(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d, n, ev, workj, lwj, info, params);
      });
      float t_copy = time_ms([&] {
        cudaMemcpyAsync(d, w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice);
      });
      // 64-bit batched SYEV with batch 1 (different small-matrix algorithm)
      cusolverDnParams_t prm;
      CK(cusolverDnCreateParams(&prm));
      size_t wd = 0, wh = 0;
      float t_evb = -1.f;
      if (cusolverDnXsyevBatched_bufferSize(sol, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                            CUDA_C_64F, d, n, CUDA_R_64F, ev, CUDA_C_64F, &wd, &wh, 1) == 0) {
        void* bd;
        cudaMalloc(&bd, wd + 16);
        std::vector<char> bh(wh + 16);
        t_evb = time_ms([&] {
          cudaMemcpyAsync(d, w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice);
          cusolverDnXsyevBatched(sol, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, d, n,
                                 CUDA_R_64F, ev, CUDA_C_64F, bd, wd, bh.data(), wh, info, 1);
        });
        cudaFree(bd);
      }
      cusolverDnDestroyParams(prm);
      printf("{\"bench\":\"eig\",\"n\":%d,\"kind\":\"%s\",\"heevd_ms\":%.3f,\"heevj_ms\":%.3f,\"syevBatched_ms\":%.3f,\"copy_ms\":%.3f}\n", n,
             kind ? "near_diag" : "random", t_evd, t_evj, t_evb, t_copy);
      cudaFree(d);
      cudaFree(w0);
      cudaFree(ev);
      cudaFree(work);
      cudaFree(workj);
      cusolverDnDestroySyevjInfo(params);
    }
  }
  // QR of an m x k panel
  for (auto mk : {std::pair<int, int>{2048, 160}, {2048, 64}, {5000, 600}, {12000, 1400}}) {
    int m = mk.first, k = mk.second;
    cuDoubleComplex *y, *y0, *tau, *g;
    cudaMalloc(&y, sizeof(cuDoubleComplex) * m * k);
    cudaMalloc(&y0, sizeof(cuDoubleComplex) * m * k);
    cudaMalloc(&tau, sizeof(cuDoubleComplex) * k);
    cudaMalloc(&g, sizeof(cuDoubleComplex) * k * k);
    std::vector<cuDoubleComplex> hy((size_t)m * k);
    for (auto& v : hy) v = make_cuDoubleComplex(nd(rng), nd(rng));
    cudaMemcpy(y0, hy.data(), sizeof(cuDoubleComplex) * m * k, cudaMemcpyHostToDevice);
    int l1 = 0, l2 = 0, l3 = 0;
    CK(cusolverDnZgeqrf_bufferSize(sol, m, k, y, m, &l1));
    CK(cusolverDnZungqr_bufferSize(sol, m, k, k, y, m, tau, &l2));
    CK(cusolverDnZpotrf_bufferSize(sol, CUBLAS_FILL_MODE_UPPER, k, g, k, &l3));
    int lw = std::max(l1, std::max(l2, l3));
    cuDoubleComplex* work;
    cudaMalloc(&work, sizeof(cuDoubleComplex) * lw);
    float t_geqrf = time_ms([&] {
      cudaMemcpyAsync(y, y0, sizeof(cuDoubleComplex) * m * k, cudaMemcpyDeviceToDevice);
      cusolverDnZgeqrf(sol, m, k, y, m, tau, work, lw, info);
    });
    float t_ungqr = time_ms([&] { cusolverDnZungqr(sol, m, k, k, y, m, tau, work, lw, info); });
    const double one = 1.0, zero = 0.0;
    const cuDoubleComplex zone = make_cuDoubleComplex(1, 0);
    float t_herk = time_ms([&] { cublasZherk(blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, k, m, &one, y0, m, &zero, g, k); });
    float t_gemm = time_ms([&] {
      const cuDoubleComplex z0 = make_cuDoubleComplex(0, 0);
      cublasZgemm(blas, CUBLAS_OP_C, CUBLAS_OP_N, k, k, m, &zone, y0, m, y0, m, &z0, g, k);
    });
    float t_potrf = time_ms([&] {
      cublasZherk(blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, k, m, &one, y0, m, &zero, g, k);
      cusolverDnZpotrf(sol, CUBLAS_FILL_MODE_UPPER, k, g, k, work, lw, info);
    }) - t_herk;
    float t_trsm = time_ms([&] {
      cublasZtrsm(blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, k, &zone, g, k, y, m);
    });
    printf("{\"bench\":\"qr\",\"m\":%d,\"k\":%d,\"geqrf_ms\":%.3f,\"ungqr_ms\":%.3f,\"herk_ms\":%.3f,\"gram_gemm_ms\":%.3f,\"potrf_ms\":%.3f,\"trsm_ms\":%.3f}\n",
           m, k, t_geqrf, t_ungqr, t_herk, t_gemm, t_potrf, t_trsm);
    cudaFree(y);
    cudaFree(y0);
    cudaFree(tau);
    cudaFree(g);
    cudaFree(work);
  }
  return 0;
}
