// Dense Hermitian eigensolvers of cuSOLVER at the Rayleigh-Ritz sizes
// (w = blk .. a few dozen): legacy zheevd, 64-bit Xsyevd, Jacobi zheevj.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 eig_bench.cu -lcusolver -o eig_bench
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__); return 1; } } while (0)

int main() {
  cusolverDnHandle_t h;
  CK(cusolverDnCreate(&h));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cusolverDnSetStream(h, s);
  cusolverDnParams_t params;
  CK(cusolverDnCreateParams(&params));
  syevjInfo_t jinfo;
  CK(cusolverDnCreateSyevjInfo(&jinfo));
  cusolverDnXsyevjSetTolerance(jinfo, 1e-15);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int n : {48, 100, 160, 200, 400, 600, 1400}) {
    std::mt19937_64 rng(n);
    std::normal_distribution<double> nd;
    std::vector<cuDoubleComplex> a((size_t)n * n);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i <= j; ++i) {
        double re = nd(rng), im = i == j ? 0.0 : nd(rng);
        a[(size_t)j * n + i] = make_cuDoubleComplex(re, im);
        a[(size_t)i * n + j] = make_cuDoubleComplex(re, -im);
      }
    cuDoubleComplex *d_a, *d_w0;
    double* d_w;
    int* d_info;
    cudaMalloc(&d_a, sizeof(cuDoubleComplex) * n * n);
    cudaMalloc(&d_w0, sizeof(cuDoubleComplex) * n * n);
    cudaMalloc(&d_w, sizeof(double) * n);
    cudaMalloc(&d_info, sizeof(int));
    cudaMemcpy(d_w0, a.data(), sizeof(cuDoubleComplex) * n * n, cudaMemcpyHostToDevice);
    const int reps = n <= 400 ? 20 : 4;
    // legacy zheevd
    int lwork = 0;
    CK(cusolverDnZheevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d_a, n, d_w, &lwork));
    cuDoubleComplex* work;
    cudaMalloc(&work, sizeof(cuDoubleComplex) * lwork);
    float t_evd = 0, t_x = 0, t_j = 0;
    for (int r = 0; r <= reps; ++r) {
      cudaMemcpyAsync(d_a, d_w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice, s);
      cudaEventRecord(e0, s);
      CK(cusolverDnZheevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d_a, n, d_w, work, lwork, d_info));
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) t_evd += ms;
    }
    // 64-bit Xsyevd
    size_t dws = 0, hws = 0;
    CK(cusolverDnXsyevd_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, d_a, n,
                                   CUDA_R_64F, d_w, CUDA_C_64F, &dws, &hws));
    void* dwork;
    cudaMalloc(&dwork, dws);
    std::vector<char> hwork(hws + 1);
    for (int r = 0; r <= reps; ++r) {
      cudaMemcpyAsync(d_a, d_w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice, s);
      cudaEventRecord(e0, s);
      CK(cusolverDnXsyevd(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, d_a, n,
                          CUDA_R_64F, d_w, CUDA_C_64F, dwork, dws, hwork.data(), hws, d_info));
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) t_x += ms;
    }
    // Jacobi
    int lj = 0;
    CK(cusolverDnZheevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d_a, n, d_w, &lj, jinfo));
    cuDoubleComplex* wj;
    cudaMalloc(&wj, sizeof(cuDoubleComplex) * lj);
    for (int r = 0; r <= reps; ++r) {
      cudaMemcpyAsync(d_a, d_w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice, s);
      cudaEventRecord(e0, s);
      CK(cusolverDnZheevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d_a, n, d_w, wj, lj, d_info, jinfo));
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) t_j += ms;
    }
    // batched API with batch 1 (CUDA 12.6+: its own small-matrix path)
    float t_b = 0;
    size_t dwb = 0, hwb = 0;
    CK(cusolverDnXsyevBatched_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F,
                                         d_a, n, CUDA_R_64F, d_w, CUDA_C_64F, &dwb, &hwb, 1));
    void* dworkb;
    cudaMalloc(&dworkb, dwb + 16);
    std::vector<char> hworkb(hwb + 1);
    for (int r = 0; r <= reps; ++r) {
      cudaMemcpyAsync(d_a, d_w0, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToDevice, s);
      cudaEventRecord(e0, s);
      CK(cusolverDnXsyevBatched(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, d_a, n,
                                CUDA_R_64F, d_w, CUDA_C_64F, dworkb, dwb, hworkb.data(), hwb, d_info, 1));
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) t_b += ms;
    }
    // residual of the batched result: max |A v - w v| over the columns
    {
      std::vector<cuDoubleComplex> v((size_t)n * n);
      std::vector<double> w(n);
      cudaMemcpy(v.data(), d_a, sizeof(cuDoubleComplex) * n * n, cudaMemcpyDeviceToHost);
      cudaMemcpy(w.data(), d_w, sizeof(double) * n, cudaMemcpyDeviceToHost);
      double worst = 0;
      for (int j = 0; j < n && n <= 400; ++j)
        for (int i = 0; i < n; ++i) {
          double re = 0, im = 0;
          for (int k = 0; k < n; ++k) {
            const cuDoubleComplex x = a[(size_t)k * n + i], y = v[(size_t)j * n + k];
            re += x.x * y.x - x.y * y.y;
            im += x.x * y.y + x.y * y.x;
          }
          re -= w[j] * v[(size_t)j * n + i].x;
          im -= w[j] * v[(size_t)j * n + i].y;
          if (fabs(re) > worst) worst = fabs(re);
          if (fabs(im) > worst) worst = fabs(im);
        }
      printf("{\"n\": %d, \"zheevd_ms\": %.3f, \"Xsyevd_ms\": %.3f, \"zheevj_ms\": %.3f, \"XsyevBatched1_ms\": %.3f,"
             " \"XsyevBatched1_resid\": %.2e}\n", n, t_evd / reps, t_x / reps, t_j / reps, t_b / reps, worst);
    }
    cudaFree(dworkb);
    cudaFree(d_a); cudaFree(d_w0); cudaFree(d_w); cudaFree(d_info); cudaFree(work); cudaFree(dwork); cudaFree(wj);
  }
  return 0;
}
