// FP64 peak microbenchmark: DFMA vs DMMA (mma.sync f64) on sm_100a.
// Measures the denominators of the FP64 roofline (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double x) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = x * (threadIdx.x + c);
  const double m = 1.0000001, a = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], m, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters, double x) {
  double a = x * threadIdx.x, b = x + threadIdx.x;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    int threads = warps * 32;
    float ms = time_it([&] { dfma_kernel<8><<<sms * 2, threads>>>(out, iters, 1.0); });
    double flops = 2.0 * 8 * iters * (double)threads * sms * 2;
    printf("{\"bench\":\"dfma\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.3f}\n", warps, sms * 2, flops / ms / 1e9);
  }
  for (int warps : {4, 8, 16}) {
    int threads = warps * 32;
    float ms = time_it([&] { dmma_kernel<8><<<sms * 2, threads>>>(out, iters / 4, 1.0); });
    double flops = 2.0 * 256 * 8 * (iters / 4) * (double)warps * sms * 2;
    printf("{\"bench\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.3f}\n", warps, sms * 2, flops / ms / 1e9);
  }
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, p.clockRate);
  return 0;
}
