// Kernels of the near-diagonal Hermitian eigensolver used by Rayleigh-Ritz
// (reference chfsi.py:347, linalg.py:181-206).
//
// After the first ChFSI loops the projected matrix G = P^H H P is close to
// diagonal: its off-diagonal entries are of the order of the Ritz residuals
// (1e-4 .. 1e-8) while the diagonal gaps are ~1e-3. One simultaneous
// first-order Jacobi step  X = I + S,  S_ij = G_ij / (d_j - d_i),  made
// unitary by Newton-Schulz polar iterations, squares the off-diagonal ratio;
// three steps reach the rounding level. All the O(w^3) work is ZGEMM on the
// tensor cores; these kernels do the O(w^2) elementwise parts. The host side
// (chfsi_abi.cu: heev_near_diag) checks convergence and falls back to
// cuSOLVER zheevd whenever the matrix is not in that regime.
#include "chfsi_internal.h"
#include "common.cuh"

namespace chfsi {

namespace {

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// max that propagates NaN (fmax drops it): a NaN anywhere must fail the checks
__device__ __forceinline__ double pmax(double a, double b) { return (b > a || isnan(b)) ? b : a; }

// X = I + S with S_ij = G_ij / (d_j - d_i); stats[0] = max_ij |G_ij| / |d_j - d_i|,
// stats[1] = max_ij |G_ij| (i != j), stats[2] = max_i |d_i|.
__global__ void nd_build_step_kernel(const double2* __restrict__ g, long long ldg, int n,
                                     double2* __restrict__ x, long long ldx, double* stats) {
  const long long total = (long long)n * n;
  double rmax = 0.0, emax = 0.0, dmax = 0.0;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx % n);
    double2 out;
    if (i == j) {
      out = make_double2(1.0, 0.0);
      dmax = pmax(dmax, fabs(g[(long long)i * ldg + i].x));
    } else {
      const double2 e = g[(long long)j * ldg + i];
      const double gap = g[(long long)j * ldg + j].x - g[(long long)i * ldg + i].x;
      const double ae = hypot(e.x, e.y);
      emax = pmax(emax, ae);
      if (ae == 0.0) {
        out = make_double2(0.0, 0.0);
      } else {
        const double ag = fabs(gap);
        rmax = pmax(rmax, ag > 0.0 ? ae / ag : INFINITY);
        out = make_double2(e.x / gap, e.y / gap);
      }
    }
    x[(long long)j * ldx + i] = out;
  }
  // block max then one atomic per block (max is order independent: exact)
  __shared__ double sh[3][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rmax = pmax(rmax, __shfl_down_sync(0xffffffffu, rmax, o));
    emax = pmax(emax, __shfl_down_sync(0xffffffffu, emax, o));
    dmax = pmax(dmax, __shfl_down_sync(0xffffffffu, dmax, o));
  }
  if (lane == 0) {
    sh[0][wid] = rmax;
    sh[1][wid] = emax;
    sh[2][wid] = dmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      rmax = pmax(rmax, sh[0][w]);
      emax = pmax(emax, sh[1][w]);
      dmax = pmax(dmax, sh[2][w]);
    }
    if (!(rmax <= 1e300)) rmax = 1e300;  // inf / nan: "not near-diagonal"
    atomic_max_nonneg(stats + 0, rmax);
    atomic_max_nonneg(stats + 1, emax);
    atomic_max_nonneg(stats + 2, dmax);
  }
}

// M = 1.5 I - 0.5 T   (Newton-Schulz polar step X <- X M with T = X^H X)
__global__ void nd_ns_matrix_kernel(double2* t, long long ldt, int n, double* defect) {
  const long long total = (long long)n * n;
  double dmax = 0.0;  // max |T - I|: the unitarity defect of the NS input
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx % n);
    double2* p = t + (long long)j * ldt + i;
    const double2 v = *p;
    dmax = pmax(dmax, hypot(v.x - (i == j ? 1.0 : 0.0), v.y));
    *p = make_double2((i == j ? 1.5 : 0.0) - 0.5 * v.x, -0.5 * v.y);
  }
  if (defect == nullptr) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = pmax(dmax, __shfl_down_sync(0xffffffffu, dmax, o));
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = dmax;
  __syncthreads();
  if (wid == 0) {
    dmax = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = pmax(dmax, __shfl_down_sync(0xffffffffu, dmax, o));
    if (lane == 0) atomic_max_nonneg(defect, dmax);
  }
}

// rank-based stable ascending sort of the real diagonal: perm[rank] = i
__global__ void nd_sort_kernel(const double2* __restrict__ g, long long ldg, int n, double* w,
                               int* perm) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double di = g[(long long)i * ldg + i].x;
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = g[(long long)j * ldg + j].x;
      rank += (dj < di) || (dj == di && j < i);
    }
    w[rank] = di;
    perm[rank] = i;
  }
}

// out[:, r] = src[:, perm[r]]
__global__ void nd_gather_cols_kernel(const double2* __restrict__ src, long long lds, int m, int n,
                                      const int* __restrict__ perm, double2* __restrict__ out,
                                      long long ldo) {
  const long long total = (long long)m * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / m), i = (int)(idx % m);
    out[(long long)r * ldo + i] = src[(long long)perm[r] * lds + i];
  }
}

inline int grid_for(long long total) {
  long long g = (total + 255) / 256;
  if (g > kNumSMs * 8) g = kNumSMs * 8;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

cudaError_t nd_build_step_launch(const double2* g, long long ldg, int n, double2* x, long long ldx,
                                 double* stats, cudaStream_t s) {
  note_launch();
  nd_build_step_kernel<<<grid_for((long long)n * n), 256, 0, s>>>(g, ldg, n, x, ldx, stats);
  return cudaGetLastError();
}

cudaError_t nd_ns_matrix_launch(double2* t, long long ldt, int n, double* defect, cudaStream_t s) {
  note_launch();
  nd_ns_matrix_kernel<<<grid_for((long long)n * n), 256, 0, s>>>(t, ldt, n, defect);
  return cudaGetLastError();
}

cudaError_t nd_sort_launch(const double2* g, long long ldg, int n, double* w, int* perm,
                           cudaStream_t s) {
  note_launch();
  nd_sort_kernel<<<(n + 127) / 128, 128, 0, s>>>(g, ldg, n, w, perm);
  return cudaGetLastError();
}

cudaError_t nd_gather_cols_launch(const double2* src, long long lds, int m, int n, const int* perm,
                                  double2* out, long long ldo, cudaStream_t s) {
  note_launch();
  nd_gather_cols_kernel<<<grid_for((long long)m * n), 256, 0, s>>>(src, lds, m, n, perm, out, ldo);
  return cudaGetLastError();
}

}  // namespace chfsi
