// Cholesky-QR pieces at the panel shapes (latency study): Gram ZGEMM,
// cuSOLVER potrf, cuBLAS ZTRSM (right), cuSOLVER Xtrtri + ZGEMM / ZTRMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 qr_bench.cu -lcublas -lcusolver -o qr_bench
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
  int shapes[][2] = {{512, 48}, {2048, 160}, {2048, 100}, {5000, 600}, {12000, 1400}, {2560, 2048}, {6000, 5000}};
  for (auto& sh : shapes) {
    const int m = sh[0], w = sh[1];
    std::mt19937_64 rng(m + w);
    std::normal_distribution<double> nd;
    std::vector<cuDoubleComplex> y((size_t)m * w);
    for (auto& v : y) v = make_cuDoubleComplex(nd(rng), nd(rng));
    cuDoubleComplex *dy, *dy2, *dg, *dg0, *dr;
    cudaMalloc(&dy, sizeof(cuDoubleComplex) * m * w);
    cudaMalloc(&dy2, sizeof(cuDoubleComplex) * m * w);
    cudaMalloc(&dg, sizeof(cuDoubleComplex) * w * w);
    cudaMalloc(&dg0, sizeof(cuDoubleComplex) * w * w);
    cudaMalloc(&dr, sizeof(cuDoubleComplex) * w * w);
    int* dinfo;
    cudaMalloc(&dinfo, sizeof(int));
    cudaMemcpy(dy, y.data(), sizeof(cuDoubleComplex) * m * w, cudaMemcpyHostToDevice);
    CK(cublasZgemm(b, CUBLAS_OP_C, CUBLAS_OP_N, w, w, m, &one, dy, m, dy, m, &zero, dg0, w));
    int lwork = 0;
    CK(cusolverDnZpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, w, dg, w, &lwork));
    cuDoubleComplex* work;
    cudaMalloc(&work, sizeof(cuDoubleComplex) * (lwork + 1));
    size_t dws = 0, hws = 0;
    CK(cusolverDnXtrtri_bufferSize(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, w, CUDA_C_64F, dr, w, &dws, &hws));
    void* dwork;
    cudaMalloc(&dwork, dws + 16);
    std::vector<char> hwork(hws + 16);
    const int reps = m <= 5000 ? 50 : 5;
    auto timeit = [&](const char* name, auto fn) {
      fn();
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) fn();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"m\":%d,\"w\":%d,\"op\":\"%s\",\"us\":%.2f}\n", m, w, name, ms * 1e3 / reps);
    };
    timeit("gram_zgemm", [&] { cublasZgemm(b, CUBLAS_OP_C, CUBLAS_OP_N, w, w, m, &one, dy, m, dy, m, &zero, dg, w); });
    timeit("gram_zherk", [&] { double o = 1, z = 0; cublasZherk(b, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, w, m, &o, dy, m, &z, dg, w); });
    timeit("copy+potrf", [&] {
      cudaMemcpyAsync(dg, dg0, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
      cusolverDnZpotrf(h, CUBLAS_FILL_MODE_UPPER, w, dg, w, work, lwork, dinfo);
    });
    {
      cuDoubleComplex** parr;
      cudaMalloc(&parr, sizeof(void*));
      cudaMemcpy(parr, &dg, sizeof(void*), cudaMemcpyHostToDevice);
      timeit("copy+potrf_batched1", [&] {
        cudaMemcpyAsync(dg, dg0, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
        cusolverDnZpotrfBatched(h, CUBLAS_FILL_MODE_UPPER, w, parr, w, dinfo, 1);
      });
      size_t xd = 0, xh = 0;
      cusolverDnXpotrf_bufferSize(h, params, CUBLAS_FILL_MODE_UPPER, w, CUDA_C_64F, dg, w, CUDA_C_64F, &xd, &xh);
      void* xw; cudaMalloc(&xw, xd + 16);
      std::vector<char> xhw(xh + 16);
      timeit("copy+xpotrf", [&] {
        cudaMemcpyAsync(dg, dg0, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
        cusolverDnXpotrf(h, params, CUBLAS_FILL_MODE_UPPER, w, CUDA_C_64F, dg, w, CUDA_C_64F, xw, xd, xhw.data(), xh, dinfo);
      });
      timeit("copy+potrf_lower", [&] {
        cudaMemcpyAsync(dg, dg0, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
        cusolverDnZpotrf(h, CUBLAS_FILL_MODE_LOWER, w, dg, w, work, lwork, dinfo);
      });
      cudaMemcpyAsync(dg, dg0, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
      cusolverDnZpotrf(h, CUBLAS_FILL_MODE_UPPER, w, dg, w, work, lwork, dinfo);
      cudaFree(xw);
    }
    // dg now holds R (upper)
    timeit("copy+trsm_right", [&] {
      cudaMemcpyAsync(dy2, dy, sizeof(cuDoubleComplex) * m * w, cudaMemcpyDeviceToDevice, s);
      cublasZtrsm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, w, &one, dg, w, dy2, m);
    });
    {  // the same solve with the LOWER factor: Y <- Y L^-H (L = R^H)
      cuDoubleComplex* dl;
      cudaMalloc(&dl, sizeof(cuDoubleComplex) * w * w);
      cudaMemcpyAsync(dl, dg0, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
      cusolverDnZpotrf(h, CUBLAS_FILL_MODE_LOWER, w, dl, w, work, lwork, dinfo);
      int hinfo = -1;
      cudaMemcpy(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
      printf("{\"m\":%d,\"w\":%d,\"op\":\"potrf_lower_info\",\"info\":%d}\n", m, w, hinfo);
      timeit("copy+trsm_right_lower_C", [&] {
        cudaMemcpyAsync(dy2, dy, sizeof(cuDoubleComplex) * m * w, cudaMemcpyDeviceToDevice, s);
        cublasZtrsm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, m, w, &one, dl, w, dy2, m);
      });
      timeit("copy+trsm_left_lower_N", [&] {  // the reduction's L^-1 A shape (m x w rhs with w x w L)
        cudaMemcpyAsync(dy2, dy, sizeof(cuDoubleComplex) * m * w, cudaMemcpyDeviceToDevice, s);
        if (m == w) cublasZtrsm(b, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, w, w, &one, dl, w, dy2, m);
      });
      cudaFree(dl);
    }
    timeit("copy_only", [&] { cudaMemcpyAsync(dy2, dy, sizeof(cuDoubleComplex) * m * w, cudaMemcpyDeviceToDevice, s); });
    timeit("copy+trtri", [&] {
      cudaMemcpyAsync(dr, dg, sizeof(cuDoubleComplex) * w * w, cudaMemcpyDeviceToDevice, s);
      cusolverDnXtrtri(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, w, CUDA_C_64F, dr, w, dwork, dws, hwork.data(), hws, dinfo);
    });
    {
      cuDoubleComplex* did;
      cudaMalloc(&did, sizeof(cuDoubleComplex) * w * w);
      std::vector<cuDoubleComplex> eye((size_t)w * w, zero);
      for (int i = 0; i < w; ++i) eye[(size_t)i * w + i] = one;
      timeit("copy+trsm_identity_w", [&] {
        cudaMemcpyAsync(did, eye.data(), 0, cudaMemcpyHostToDevice, s);
        cublasZtrsm(b, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, w, w, &one, dg, w, did, w);
      });
      timeit("trmm_inplace", [&] { cublasZtrmm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, w, &one, dr, w, dy2, m, dy2, m); });
      cudaFree(did);
    }
    timeit("gemm_y_rinv", [&] { cublasZgemm(b, CUBLAS_OP_N, CUBLAS_OP_N, m, w, w, &one, dy, m, dr, w, &zero, dy2, m); });
    timeit("trmm_y_rinv", [&] { cublasZtrmm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, w, &one, dr, w, dy, m, dy2, m); });
    cudaFree(dy); cudaFree(dy2); cudaFree(dg); cudaFree(dg0); cudaFree(dr); cudaFree(work); cudaFree(dwork);
  }
  return 0;
}
