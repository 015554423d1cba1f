// Shared device helpers for the ChFSI sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace chfsi {



// ---- cp.async (LDGSTS): 16-byte global->shared copy with zero fill -------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- FP64 tensor core: DMMA.8x8x4 (the native sm_100a f64 MMA) ----------
// A 8x4 row fragment: lane (g = lane/4, t = lane%4) holds A[g][t].
// B 4x8 col fragment: lane holds B[t][g].
// C 8x8: lane holds C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 lds128(const unsigned char* p) {
  return *reinterpret_cast<const double2*>(p);
}

// Round-to-nearest, never contracted into FMA: keeps the epilogue arithmetic
// in the same operation order as the reference's numpy expression.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

}  // namespace chfsi
