// Reduction to standard form H = L^-1 A L^-H (B = L L^H) at the BASELINE n:
//   (a) potrf + ZTRSM(left, L) + ZTRSM(right, L^H)          (the current path)
//   (b) potrf + Xtrtri(L) + ZTRMM(left, L^-1) + ZTRMM(right, L^-H), out of place
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 reduce_bench.cu -lcublas -lcusolver -o reduce_bench
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdio>
#include <vector>

#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__); return 1; } } while (0)

__global__ void fill_hpd(cuDoubleComplex* a, int n, unsigned seed, double diag) {
  long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    int j = (int)(e / n), i = (int)(e % n);
    int lo = i < j ? i : j, hi = i < j ? j : i;
    unsigned h = (unsigned)(lo * 2654435761u) ^ (unsigned)(hi * 40503u) ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    double re = ((h & 0xffff) / 65536.0 - 0.5) / n, im = (((h >> 16) & 0xffff) / 65536.0 - 0.5) / n;
    if (i == j) { re = diag; im = 0; }
    a[e] = make_cuDoubleComplex(re, i < j ? im : -im);
  }
}

int main() {
  cublasHandle_t b;
  cusolverDnHandle_t h;
  CK(cublasCreate(&b));
  CK(cusolverDnCreate(&h));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cublasSetStream(b, s);
  cusolverDnSetStream(h, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const cuDoubleComplex one = make_cuDoubleComplex(1, 0);
  for (int n : {2048, 5000, 12000}) {
    size_t bytes = sizeof(cuDoubleComplex) * (size_t)n * n;
    cuDoubleComplex *A0, *A, *B0, *L, *W, *T;
    CK(cudaMalloc(&A0, bytes)); CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B0, bytes));
    CK(cudaMalloc(&L, bytes)); CK(cudaMalloc(&W, bytes)); CK(cudaMalloc(&T, bytes));
    fill_hpd<<<1184, 256, 0, s>>>(A0, n, 1u, 3.0);
    fill_hpd<<<1184, 256, 0, s>>>(B0, n, 7u, 1.5);
    int* info; cudaMalloc(&info, sizeof(int));
    int lwork = 0;
    CK(cusolverDnZpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, L, n, &lwork));
    cuDoubleComplex* work; CK(cudaMalloc(&work, sizeof(cuDoubleComplex) * (lwork + 1)));
    cusolverDnParams_t params; cusolverDnCreateParams(&params);
    size_t dws = 0, hws = 0;
    CK(cusolverDnXtrtri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_C_64F, W, n, &dws, &hws));
    void* dwork; CK(cudaMalloc(&dwork, dws + 16));
    std::vector<char> hwork(hws + 16);
    auto timeit = [&](const char* name, auto prep, auto fn) {
      float tot = 0; int reps = n <= 5000 ? 5 : 2;
      for (int r = 0; r <= reps; ++r) {
        prep();
        cudaEventRecord(e0, s); fn(); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) tot += ms;
      }
      printf("{\"n\":%d,\"op\":\"%s\",\"ms\":%.3f}\n", n, name, tot / reps);
    };
    auto prepL = [&] { cudaMemcpyAsync(L, B0, bytes, cudaMemcpyDeviceToDevice, s); };
    timeit("potrf_lower", prepL, [&] { cusolverDnZpotrf(h, CUBLAS_FILL_MODE_LOWER, n, L, n, work, lwork, info); });
    // L holds the factor now (strict upper is garbage/ignored)
    auto prepA = [&] { cudaMemcpyAsync(A, A0, bytes, cudaMemcpyDeviceToDevice, s); };
    timeit("trsm_left_N", prepA, [&] { cublasZtrsm(b, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n, &one, L, n, A, n); });
    timeit("trsm_right_C", [] {}, [&] { cublasZtrsm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, n, n, &one, L, n, A, n); });
    auto prepW = [&] { cudaMemcpyAsync(W, L, bytes, cudaMemcpyDeviceToDevice, s); };
    timeit("trtri_lower", prepW, [&] { cusolverDnXtrtri(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_C_64F, W, n, dwork, dws, hwork.data(), hws, info); });
    timeit("trmm_left_N", [] {}, [&] { cublasZtrmm(b, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n, &one, W, n, A0, n, T, n); });
    timeit("trmm_right_C", [] {}, [&] { cublasZtrmm(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, n, n, &one, W, n, T, n, A, n); });
    timeit("zgemm_nn", [] {}, [&] { cublasZgemm(b, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, W, n, A0, n, &one, T, n); });
    cudaFree(A0); cudaFree(A); cudaFree(B0); cudaFree(L); cudaFree(W); cudaFree(T); cudaFree(work); cudaFree(dwork);
  }
  return 0;
}
