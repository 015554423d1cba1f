// Grid-wide barrier latency on a B200: cooperative_groups grid.sync() vs a
// hand-written sense-reversing barrier (one atomicAdd per CTA, everyone polls
// a generation word with ld.acquire), cooperative launch, 256 threads/CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -rdc=false grid_barrier.cu -o grid_barrier
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group grid = cg::this_grid();
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    v = v * 1.0000001 + 1.0;
    grid.sync();
  }
  if (v == -1.0) *sink = v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// bar[0] = arrival counter, bar[32] = generation (separate 128-byte lines)
__device__ __forceinline__ void own_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned next = gen + 1;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(bar + 32), "r"(next) : "memory");
    } else {
      while (ld_acquire(bar + 32) != next) {
      }
    }
  }
  gen += 1;
  __syncthreads();
}

__global__ void k_own(int iters, unsigned* bar, unsigned gen0, double* sink) {
  double v = threadIdx.x;
  unsigned gen = gen0;
  for (int i = 0; i < iters; ++i) {
    v = v * 1.0000001 + 1.0;
    own_barrier(bar, gen);
  }
  if (v == -1.0) *sink = v;
}

int main() {
  double* sink;
  unsigned* bar;
  cudaMalloc(&sink, 8);
  cudaMalloc(&bar, 256);
  cudaMemset(bar, 0, 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  unsigned gen = 0;
  for (int grid : {32, 100, 148, 296}) {
    float ms_cg = 0, ms_own = 0;
    for (int rep = 0; rep < 3; ++rep) {
      int it = iters;
      void* a1[] = {&it, &sink};
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k_cg, dim3(grid), dim3(256), a1, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms_cg, e0, e1);
      void* a2[] = {&it, &bar, &gen, &sink};
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k_own, dim3(grid), dim3(256), a2, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms_own, e0, e1);
      gen += iters;
    }
    printf("{\"grid\": %d, \"cg_grid_sync_us\": %.2f, \"own_barrier_us\": %.2f, \"err\": \"%s\"}\n", grid,
           ms_cg * 1e3 / iters, ms_own * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
