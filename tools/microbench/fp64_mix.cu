// Does DMMA share the FP64 pipe with DFMA/DADD on sm_100a?  Decides the
// complex-product formulation of K1: the 3M (Gauss) product trades 1 of 4
// DMMAs per complex block for DADDs that form the operand sums.
//   dmma only:            D DMMA.8x8x4 per iteration
//   dmma + dfma:          D DMMA + F independent DFMA per iteration
// If the pipes are separate, the mixed time ~= max(dmma, dfma); if shared,
// ~= sum.
#include <cstdio>
#include <cuda_runtime.h>

template <int D, int F>
__global__ void mix_kernel(double* out, int iters, double x) {
  double a = x * threadIdx.x, b = x + threadIdx.x;
  double c[D > 0 ? D : 1][2];
  double f[F > 0 ? F : 1];
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : 1); ++k) { c[k][0] = 0; c[k][1] = 0; }
#pragma unroll
  for (int k = 0; k < (F > 0 ? F : 1); ++k) f[k] = x * (threadIdx.x + k);
  const double m = 1.0000001, ad = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < D; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int k = 0; k < F; ++k) f[k] = fma(f[k], m, ad);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) s += c[k][0] + c[k][1];
#pragma unroll
  for (int k = 0; k < F; ++k) s += f[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename Fn>
float time_it(Fn fn) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  fn(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

template <int D, int F>
void run(int sms, double* out, int iters) {
  const int threads = 256, ctas = sms * 2;
  float ms = time_it([&] { mix_kernel<D, F><<<ctas, threads>>>(out, iters, 1.0); });
  double warps = (double)ctas * threads / 32;
  double dmma_flops = 2.0 * 256 * D * iters * warps;
  double dfma_flops = 2.0 * F * iters * warps * 32;
  printf("{\"bench\":\"mix\",\"dmma_per_iter\":%d,\"dfma_per_iter\":%d,\"ms\":%.4f,"
         "\"dmma_tflops\":%.3f,\"dfma_tflops\":%.3f,\"total_tflops\":%.3f}\n",
         D, F, ms, dmma_flops / ms / 1e9, dfma_flops / ms / 1e9, (dmma_flops + dfma_flops) / ms / 1e9);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  const int iters = 4000;
  run<12, 0>(sms, out, iters);
  run<16, 0>(sms, out, iters);
  run<0, 32>(sms, out, iters);
  run<12, 4>(sms, out, iters);   // 3M inner step: 12 DMMA + 4 operand-sum adds
  run<12, 8>(sms, out, iters);
  run<8, 64>(sms, out, iters);   // equal DMMA / DFMA flops: 8*512 vs 64*64
  run<8, 32>(sms, out, iters);
  return 0;
}
