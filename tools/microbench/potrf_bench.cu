// Small Hermitian Cholesky latency at the Rayleigh-Ritz / Cholesky-QR panel
// widths: cusolverDnZpotrf (lower), cusolverDnXpotrf, cusolverDnZpotrfBatched
// (batch 1), and ZTRSM right (the Cholesky-QR pass-1 solve), CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 potrf_bench.cu -lcublas -lcusolver -o potrf_bench
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdio>
#include <random>
#include <vector>

#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__); return 1; } } while (0)

int main() {
  cublasHandle_t b;
  cusolverDnHandle_t h;
  CK(cublasCreate(&b));
  CK(cusolverDnCreate(&h));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cublasSetStream(b, s);
  cusolverDnSetStream(h, s);
  cusolverDnParams_t params;
  CK(cusolverDnCreateParams(&params));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
  const int ws[] = {48, 100, 160, 200, 300, 600};
  const int m = 2048;
  for (int w : ws) {
    std::mt19937_64 rng(w);
    std::normal_distribution<double> nd;
    std::vector<cuDoubleComplex> y((size_t)m * w);
    for (auto& v : y) v = make_cuDoubleComplex(nd(rng), nd(rng));
    cuDoubleComplex *dy, *dg, *dg0;
    cudaMalloc(&dy, sizeof(cuDoubleComplex) * m * w);
    cudaMalloc(&dg, sizeof(cuDoubleComplex) * w * w);
    cudaMalloc(&dg0, sizeof(cuDoubleComplex) * w * w);
    int* dinfo;
    cudaMalloc(&dinfo, sizeof(int));
    cudaMemcpy(dy, y.data(), sizeof(cuDoubleComplex) * m * w, cudaMemcpyHostToDevice);
    CK(cublasZgemm(b, CUBLAS_OP_C, CUBLAS_OP_N, w, w, m, &one, dy, m, dy, m, &zero, dg0, w));
    int lwork = 0;
    CK(cusolverDnZpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, w, dg, w, &lwork));
    cuDoubleComplex* work;
    cudaMalloc(&work, sizeof(cuDoubleComplex) * (lwork + 1));
    size_t dws = 0, hws = 0;
    CK(cusolverDnXpotrf_bufferSize(h, params, CUBLAS_FILL_MODE_LOWER, w, CUDA_C_64F, dg, w,
                                   CUDA_C_64F, &dws, &hws));
    void* dwork;
    cudaMalloc(&dwork, dws + 16);
    std::vector<char> hwork(hws + 16);
    cuDoubleComplex** darr;
    cudaMalloc(&darr, sizeof(void*));
    cudaMemcpy(darr, &dg, sizeof(void*), cudaMemcpyHostToDevice);
    const int reps = 50;
    auto timeit = [&](const char* name, auto fn) {
      fn();
      cudaStreamSynchronize(s);
      float total = 0.f;
      for (int r = 0; r < reps; ++r) {
        cudaMemcpyAsync(dg, dg0, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
        cudaEventRecord(e0, s);
        fn();
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        total += ms;
      }
      printf("w=%4d %-28s %8.1f us\n", w, name, 1e3f * total / reps);
      return 0;
    };
    timeit("Zpotrf lower", [&] {
      cusolverDnZpotrf(h, CUBLAS_FILL_MODE_LOWER, w, dg, w, work, lwork, dinfo);
    });
    timeit("Xpotrf lower", [&] {
      cusolverDnXpotrf(h, params, CUBLAS_FILL_MODE_LOWER, w, CUDA_C_64F, dg, w, CUDA_C_64F, dwork,
                       dws, hwork.data(), hws, dinfo);
    });
    timeit("ZpotrfBatched(1) lower", [&] {
      cusolverDnZpotrfBatched(h, CUBLAS_FILL_MODE_LOWER, w, darr, w, dinfo, 1);
    });
    timeit("ZtrsmR (2048 x w)", [&] {
      cublasZtrsm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, m, w,
                  &one, dg0, w, dy, m);
    });
    timeit("Gram ZGEMM (w x w x 2048)", [&] {
      cublasZgemm(b, CUBLAS_OP_C, CUBLAS_OP_N, w, w, m, &one, dy, m, dy, m, &zero, dg, w);
    });
    timeit("ZGEMM w^3", [&] {
      cublasZgemm(b, CUBLAS_OP_N, CUBLAS_OP_N, w, w, w, &one, dg0, w, dg0, w, &zero, dg, w);
    });
    cudaFree(dy); cudaFree(dg); cudaFree(dg0); cudaFree(work); cudaFree(dwork); cudaFree(darr);
  }
  return 0;
}
