// Auxiliary sm_100a kernels on the ChFSI path: the Lanczos chain (K2), the
// column residual norms of Rayleigh-Ritz (K4), the Hermitian symmetrize /
// defect checks of the reduction (K5) and small layout helpers.
//
// Every reduction uses a fixed partition and a fixed combining tree, so all
// results are bitwise run-to-run reproducible (no float atomics); max-type
// reductions use integer atomics on non-negative doubles, which is exact.
#include "chfsi_internal.h"
#include "common.cuh"

namespace chfsi {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;  // valid in lane 0
}

__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Fixed-tree block sum; result valid in thread 0. blockDim.x multiple of 32, <= 1024.
__device__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

__device__ double2 block_sum2(double2 v, double2* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum2(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  if (wid == 0) {
    r = lane < nw ? sh[lane] : make_double2(0.0, 0.0);
    r = warp_sum2(r);
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ bool is_done(const int* done) { return done != nullptr && *done; }

// ------------------------------------------------------------- GEMV (K2) ---
// One warp per row; 16-byte coalesced row reads; fixed lane-strided order.
template <bool CONJ>
__global__ void gemv_rows_kernel(const double2* __restrict__ h, long long ldh,
                                 const double2* __restrict__ q, double2* __restrict__ u, int n,
                                 int rows, const int* done) {
  if (is_done(done)) return;
  const int lane = threadIdx.x & 31;
  const int warps = (blockDim.x >> 5) * gridDim.x;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
    const double2* hr = h + (long long)row * ldh;
    double sr = 0.0, si = 0.0;
    int k = lane;
    for (; k + 96 < n; k += 128) {
      double2 a0 = hr[k], a1 = hr[k + 32], a2 = hr[k + 64], a3 = hr[k + 96];
      double2 b0 = q[k], b1 = q[k + 32], b2 = q[k + 64], b3 = q[k + 96];
      const double s = CONJ ? -1.0 : 1.0;
      sr = fma(a0.x, b0.x, fma(-s * a0.y, b0.y, sr));
      si = fma(a0.x, b0.y, fma(s * a0.y, b0.x, si));
      sr = fma(a1.x, b1.x, fma(-s * a1.y, b1.y, sr));
      si = fma(a1.x, b1.y, fma(s * a1.y, b1.x, si));
      sr = fma(a2.x, b2.x, fma(-s * a2.y, b2.y, sr));
      si = fma(a2.x, b2.y, fma(s * a2.y, b2.x, si));
      sr = fma(a3.x, b3.x, fma(-s * a3.y, b3.y, sr));
      si = fma(a3.x, b3.y, fma(s * a3.y, b3.x, si));
    }
    for (; k < n; k += 32) {
      const double2 a = hr[k], b = q[k];
      const double s = CONJ ? -1.0 : 1.0;
      sr = fma(a.x, b.x, fma(-s * a.y, b.y, sr));
      si = fma(a.x, b.y, fma(s * a.y, b.x, si));
    }
    sr = warp_sum(sr);
    si = warp_sum(si);
    if (lane == 0) u[row] = make_double2(sr, si);
  }
}

// ------------------------------------------------- deterministic reductions ---
// op 0: Re(x^H y); op 1: |x|^2
template <int OP>
__global__ void reduce_partial_kernel(const double2* __restrict__ x, const double2* __restrict__ y,
                                      long long n, double* __restrict__ partial, const int* done) {
  __shared__ double sh[32];
  if (is_done(done)) return;
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x[i];
    if (OP == 0) {
      const double2 b = y[i];
      acc = fma(a.x, b.x, fma(a.y, b.y, acc));
    } else {
      acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

template <int OP>
__global__ void reduce_final_kernel(const double* __restrict__ partial, int np, double* out,
                                    const int* done) {
  __shared__ double sh[32];
  if (is_done(done)) return;
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partial[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) *out = OP == 1 ? sqrt(acc) : acc;  // OP 2: sum of squares
}

__global__ void sqrt_scalar_kernel(double* x) { *x = sqrt(*x); }

// dst = src and *out = ||src||_2 in ONE launch (the Cholesky-QR's backup copy
// and Frobenius norm): every block copies its grid-stride slice and leaves
// its partial sum of squares; the block that takes the last ticket adds the
// partials in block order (fixed: bitwise reproducible) and re-arms the counter.
__global__ void __launch_bounds__(kRedThreads) copy_norm2_kernel(const double2* __restrict__ src,
                                                                 double2* __restrict__ dst, long long n,
                                                                 double* __restrict__ partial,
                                                                 unsigned* counter, double* out) {
  __shared__ double sh[32];
  __shared__ bool last;
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {  // four independent loads per trip
    double2 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      dst[i + u * stride] = a[u];
      acc = fma(a[u].x, a[u].x, fma(a[u].y, a[u].y, acc));
    }
  }
  for (; i < n; i += stride) {
    const double2 a = src[i];
    dst[i] = a;
    acc = fma(a.x, a.x, fma(a.y, a.y, acc));
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = acc;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double tot = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) tot += __ldcg(partial + i);
  tot = block_sum(tot, sh);
  if (threadIdx.x == 0) {
    *out = sqrt(tot);
    *counter = 0u;
  }
}

// out[j] = V[:,j]^H r, one block per column
__global__ void colsdot_kernel(const double2* __restrict__ v, long long ldv, int n,
                               const double2* __restrict__ r, double2* __restrict__ out,
                               const int* done) {
  __shared__ double2 sh[32];
  if (is_done(done)) return;
  const int j = blockIdx.x;
  const double2* col = v + (long long)j * ldv;
  double2 acc = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 a = col[i], b = r[i];
    acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));   // Re(conj(a) b)
    acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));  // Im(conj(a) b)
  }
  acc = block_sum2(acc, sh);
  if (threadIdx.x == 0) out[j] = acc;
}

// r[i] -= sum_j V[i,j] coef[j]
__global__ void sub_vcoef_kernel(const double2* __restrict__ v, long long ldv, int n, int ncols,
                                 const double2* __restrict__ coef, double2* __restrict__ r,
                                 const int* done) {
  if (is_done(done)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sr = 0.0, si = 0.0;
  for (int j = 0; j < ncols; ++j) {
    const double2 a = v[(long long)j * ldv + i], c = coef[j];
    sr = fma(a.x, c.x, fma(-a.y, c.y, sr));
    si = fma(a.x, c.y, fma(a.y, c.x, si));
  }
  const double2 ri = r[i];
  r[i] = make_double2(ri.x - sr, ri.y - si);
}

// r = (u - alpha q) - beta_prev qprev
__global__ void lanczos_residual_kernel(const double2* __restrict__ u, const double2* __restrict__ q,
                                        const double2* __restrict__ qprev,
                                        const double* alpha_i, const double* beta_prev,
                                        double2* __restrict__ r, int n, const int* done) {
  if (is_done(done)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = *alpha_i;
  const double2 ui = u[i], qi = q[i];
  double rr = dsub(ui.x, dmul(a, qi.x)), ri = dsub(ui.y, dmul(a, qi.y));
  if (qprev != nullptr) {
    const double b = *beta_prev;
    const double2 p = qprev[i];
    rr = dsub(rr, dmul(b, p.x));
    ri = dsub(ri, dmul(b, p.y));
  }
  r[i] = make_double2(rr, ri);
}

// Breakdown test (chfsi.py:152) and q_{i+1} = r / beta.
__global__ void lanczos_advance_kernel(const double2* __restrict__ r, const double* beta,
                                       double2* __restrict__ qnext, double* betas_i,
                                       LanczosState* st, int i, int k, int n) {
  if (st->done) return;
  const double b = *beta;
  const bool stop = (b < 1e-14) || (i == k - 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->steps = i + 1;
    st->beta_last = b;
    if (stop) st->done = 1;
    else *betas_i = b;
  }
  if (stop) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n) {
    const double2 x = r[idx];
    qnext[idx] = make_double2(__ddiv_rn(x.x, b), __ddiv_rn(x.y, b));
  }
}

// ----------------------------------------------------- Rayleigh-Ritz (K4) ---
__global__ void colnorm_residual_kernel(const double2* __restrict__ hp, long long ldhp,
                                        const double2* __restrict__ p, long long ldp,
                                        const double* __restrict__ lambda, int n,
                                        double* __restrict__ res, int squared) {
  __shared__ double sh[32];
  const int j = blockIdx.x;
  const double lam = lambda ? lambda[j] : 0.0;
  const double2* a = hp + (long long)j * ldhp;
  const double2* b = p ? p + (long long)j * ldp : nullptr;
  double acc = 0.0;
  // (four rows per trip, their loads issued together: the one-row loop
  // serialised an L2 latency per trip; same summation order per thread)
  int i = threadIdx.x;
  for (; i + 3 * (int)blockDim.x < n; i += 4 * blockDim.x) {
    double2 x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = a[i + u * blockDim.x];
    if (b) {
#pragma unroll
      for (int u = 0; u < 4; ++u) y[u] = b[i + u * blockDim.x];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (b) {
        x[u].x = dsub(x[u].x, dmul(lam, y[u].x));
        x[u].y = dsub(x[u].y, dmul(lam, y[u].y));
      }
      acc = fma(x[u].x, x[u].x, fma(x[u].y, x[u].y, acc));
    }
  }
  for (; i < n; i += blockDim.x) {
    double2 x = a[i];
    if (b) {
      const double2 y = b[i];
      x.x = dsub(x.x, dmul(lam, y.x));
      x.y = dsub(x.y, dmul(lam, y.y));
    }
    acc = fma(x.x, x.x, fma(x.y, x.y, acc));
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) res[j] = squared ? acc : sqrt(acc);
}

// -------------------------------------------------- Hermitian helpers (K5) ---
constexpr int TS = 32;

__global__ void symmetrize_kernel(double2* a, long long lda, int n) {
  __shared__ double2 t1[TS][TS + 1];
  __shared__ double2 t2[TS][TS + 1];
  const int bi = blockIdx.y, bj = blockIdx.x;  // tile (row block bi, col block bj), bi >= bj
  if (bi < bj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // load tile (bi, bj) as t1[r][c] and tile (bj, bi) as t2[r][c] (col-major: row fastest)
  for (int c = ty; c < TS; c += 8) {
    const int r1 = bi * TS + tx, c1 = bj * TS + c;
    if (r1 < n && c1 < n) t1[tx][c] = a[(long long)c1 * lda + r1];
    const int r2 = bj * TS + tx, c2 = bi * TS + c;
    if (r2 < n && c2 < n) t2[tx][c] = a[(long long)c2 * lda + r2];
  }
  __syncthreads();
  for (int c = ty; c < TS; c += 8) {
    // element (r1, c1) = (bi*TS+tx, bj*TS+c) pairs with (c1, r1) = t2[c][tx]
    const int r1 = bi * TS + tx, c1 = bj * TS + c;
    if (r1 < n && c1 < n) {
      double2 x = t1[tx][c];
      const double2 y = t2[c][tx];
      double2 out;
      if (r1 == c1) out = make_double2(x.x, 0.0);
      else out = make_double2((x.x + y.x) * 0.5, (x.y - y.y) * 0.5);
      a[(long long)c1 * lda + r1] = out;
    }
  }
  if (bi == bj) return;
  for (int c = ty; c < TS; c += 8) {
    const int r2 = bj * TS + tx, c2 = bi * TS + c;
    if (r2 < n && c2 < n) {
      const double2 x = t2[tx][c];   // (r2, c2)
      const double2 y = t1[c][tx];   // (c2, r2)
      a[(long long)c2 * lda + r2] = make_double2((x.x + y.x) * 0.5, (x.y - y.y) * 0.5);
    }
  }
}

__global__ void herm_defect_kernel(const double2* __restrict__ a, long long lda, int n,
                                   unsigned long long* out) {
  __shared__ double2 t2[TS][TS + 1];
  __shared__ double smax[2][8];
  const int bi = blockIdx.y, bj = blockIdx.x;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int c = ty; c < TS; c += 8) {
    const int r2 = bj * TS + tx, c2 = bi * TS + c;
    if (r2 < n && c2 < n) t2[tx][c] = a[(long long)c2 * lda + r2];
  }
  __syncthreads();
  double dmax = 0.0, amax = 0.0;
  for (int c = ty; c < TS; c += 8) {
    const int r1 = bi * TS + tx, c1 = bj * TS + c;
    if (r1 < n && c1 < n) {
      const double2 x = a[(long long)c1 * lda + r1];
      const double2 y = t2[c][tx];
      dmax = fmax(dmax, hypot(x.x - y.x, x.y + y.y));
      amax = fmax(amax, hypot(x.x, x.y));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_down_sync(0xffffffffu, dmax, o));
    amax = fmax(amax, __shfl_down_sync(0xffffffffu, amax, o));
  }
  if (tx == 0) {
    smax[0][ty] = dmax;
    smax[1][ty] = amax;
  }
  __syncthreads();
  if (tx == 0 && ty == 0) {
    for (int i = 1; i < 8; ++i) {
      dmax = fmax(dmax, smax[0][i]);
      amax = fmax(amax, smax[1][i]);
    }
    atomicMax(out + 0, (unsigned long long)__double_as_longlong(dmax));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(amax));
  }
}

// dst = src^H (n x n, column-major both), tiled through shared memory
__global__ void conj_transpose_kernel(const double2* src, long long lds, double2* dst, long long ldd,
                                      int n) {
  __shared__ double2 t[TS][TS + 1];
  const int bi = blockIdx.y, bj = blockIdx.x;  // source tile (row block bi, col block bj)
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int c = ty; c < TS; c += 8) {
    const int r = bi * TS + tx, col = bj * TS + c;
    if (r < n && col < n) t[tx][c] = src[(long long)col * lds + r];
  }
  __syncthreads();
  // dst tile (bj, bi): dst[r'][c'] = conj(src[c'][r'])
  for (int c = ty; c < TS; c += 8) {
    const int r = bj * TS + tx, col = bi * TS + c;
    if (r < n && col < n) {
      const double2 v = t[c][tx];
      dst[(long long)col * ldd + r] = make_double2(v.x, -v.y);
    }
  }
}

__global__ void conj_inplace_kernel(double2* a, long long lda, int m, int n) {
  const long long total = (long long)m * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx / m, i = idx % m;
    double2* p = a + j * lda + i;
    p->y = -p->y;
  }
}

__global__ void zero_upper_kernel(double2* a, long long lda, int n) {
  const long long total = (long long)n * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx / n, i = idx % n;
    if (i < j) a[j * lda + i] = make_double2(0.0, 0.0);
  }
}

__global__ void phase_fix_kernel(double2* q, long long ldq, int m, int n,
                                 const double2* __restrict__ rdiag) {
  const long long total = (long long)m * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx / m, i = idx % m;
    const double2 d = rdiag[j];
    const double ad = hypot(d.x, d.y);
    const double pr = __ddiv_rn(d.x, ad), pi = -__ddiv_rn(d.y, ad);  // conj(d/|d|)
    double2* p = q + j * ldq + i;
    const double2 x = *p;
    *p = make_double2(dsub(dmul(x.x, pr), dmul(x.y, pi)), dadd(dmul(x.x, pi), dmul(x.y, pr)));
  }
}

__global__ void extract_diag_kernel(const double2* a, long long lda, int n, double2* diag) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) diag[j] = a[(long long)j * lda + j];
}

__global__ void copy_cols_kernel(const double2* __restrict__ x, long long ldx,
                                 double2* __restrict__ y, long long ldy, int m, int n) {
  const long long total = (long long)m * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx / m, i = idx % m;
    y[j * ldy + i] = x[j * ldx + i];
  }
}

__global__ void div_scalar_kernel(const double2* __restrict__ x, const double* d,
                                  double2* __restrict__ y, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double b = *d;
    const double2 v = x[i];
    y[i] = make_double2(__ddiv_rn(v.x, b), __ddiv_rn(v.y, b));
  }
}

__global__ void add_diag_shift_kernel(double2* a, long long lda, int n, const double* fro,
                                      double coef) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double f = *fro;
    a[(long long)i * lda + i].x += coef * f * f;
  }
}

__global__ void diag_accumulate_kernel(const double2* r, long long ldr, int n, double* acc,
                                       int first) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) acc[i] = (first ? 1.0 : acc[i]) * r[(long long)i * ldr + i].x;
}

// Second Cholesky-QR pass linearised (see chfsi_internal.h): G = I + E in,
// M = I - tri(E) out (in place, upper triangle; strict lower zeroed), where
// tri(E) = strict-upper(E) + diag(E)/2, so Q1 M has Q^H Q = I + O(|E|^2).
// out[0] = max |E_ij| (NaN propagates), acc[i] *= 1 + E_ii/2 (~ R2_ii),
// last[i] = 1 + E_ii/2. One block: the matrix is at most a few hundred wide.
constexpr int kNiThreads = 1024;
__global__ void __launch_bounds__(kNiThreads) near_identity_update_kernel(
    double2* g, long long ldg, int n, double* acc, double* last, double* out) {
  __shared__ double red[kNiThreads / 32];
  double emax = 0.0;
  const long long total = (long long)n * n;
  for (long long e = threadIdx.x; e < total; e += kNiThreads) {
    const int j = (int)(e / n), i = (int)(e - (long long)j * n);  // column-major (i, j)
    double2* p = g + (long long)j * ldg + i;
    if (i > j) {
      *p = make_double2(0.0, 0.0);
      continue;
    }
    const double2 v = *p;
    if (i == j) {
      const double d = v.x - 1.0, m = fmax(fabs(d), fabs(v.y));
      emax = (m > emax || m != m) ? m : emax;
      const double r2 = 1.0 + 0.5 * d;
      acc[i] *= r2;
      last[i] = r2;
      *p = make_double2(1.0 - 0.5 * d, 0.0);
    } else {
      const double m = fmax(fabs(v.x), fabs(v.y));
      emax = (m > emax || m != m) ? m : emax;
      *p = make_double2(-v.x, -v.y);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_down_sync(0xffffffffu, emax, o);
    emax = (t > emax || t != t) ? t : emax;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < kNiThreads / 32; ++w) m = (red[w] > m || red[w] != red[w]) ? red[w] : m;
    out[0] = m;
  }
}

// First Chebyshev step from a known product HY = H Y0 (columns j of n x w
// blocks): Y1 = alpha (HY - c Y0), K1's epilogue arithmetic in the same
// order (the step has no Yprev term).
__global__ void cheb_first_step_kernel(const double2* hy, long long ldhy, const double2* y0,
                                       long long ldy, double2* out, long long ldo, int n, int w,
                                       double alpha, double c) {
  const long long total = (long long)n * w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / n), i = (int)(e - (long long)j * n);
    const double2 a = hy[(long long)j * ldhy + i], y = y0[(long long)j * ldy + i];
    double tr = a.x, ti = a.y;
    if (c != 0.0) {
      tr = __dsub_rn(tr, __dmul_rn(c, y.x));
      ti = __dsub_rn(ti, __dmul_rn(c, y.y));
    }
    out[(long long)j * ldo + i] = make_double2(__dmul_rn(alpha, tr), __dmul_rn(alpha, ti));
  }
}

inline int grid_for(long long total, int threads, int cap = kNumSMs * 16) {
  long long g = (total + threads - 1) / threads;
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

cudaError_t gemv_rows_launch(const double2* h, long long ldh, bool conj_h, const double2* q,
                             double2* u, int n, const int* done, cudaStream_t s, int rows) {
  if (rows < 0) rows = n;
  const int threads = 256;
  const int blocks = grid_for((long long)rows * 32, threads, kNumSMs * 8);
  note_launch();
  if (conj_h) gemv_rows_kernel<true><<<blocks, threads, 0, s>>>(h, ldh, q, u, n, rows, done);
  else gemv_rows_kernel<false><<<blocks, threads, 0, s>>>(h, ldh, q, u, n, rows, done);
  return cudaGetLastError();
}

cudaError_t dot_re_launch(const double2* x, const double2* y, int n, double* partial, double* out,
                          const int* done, cudaStream_t s) {
  note_launch();
  reduce_partial_kernel<0><<<kRedBlocks, kRedThreads, 0, s>>>(x, y, n, partial, done);
  note_launch();
  reduce_final_kernel<0><<<1, 1024, 0, s>>>(partial, kRedBlocks, out, done);
  return cudaGetLastError();
}

cudaError_t norm2_launch(const double2* x, long long n, double* partial, double* out,
                         const int* done, cudaStream_t s) {
  note_launch();
  reduce_partial_kernel<1><<<kRedBlocks, kRedThreads, 0, s>>>(x, nullptr, n, partial, done);
  note_launch();
  reduce_final_kernel<1><<<1, 1024, 0, s>>>(partial, kRedBlocks, out, done);
  return cudaGetLastError();
}

cudaError_t copy_norm2_launch(const double2* src, double2* dst, long long n, double* partial,
                              unsigned* counter, double* out, cudaStream_t s) {
  note_launch();
  copy_norm2_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(src, dst, n, partial, counter, out);
  return cudaGetLastError();
}

cudaError_t norm2sq_launch(const double2* x, long long n, double* partial, double* out,
                           const int* done, cudaStream_t s) {
  note_launch();
  reduce_partial_kernel<1><<<kRedBlocks, kRedThreads, 0, s>>>(x, nullptr, n, partial, done);
  note_launch();
  reduce_final_kernel<2><<<1, 1024, 0, s>>>(partial, kRedBlocks, out, done);
  return cudaGetLastError();
}

cudaError_t sqrt_scalar_launch(double* x, cudaStream_t s) {
  note_launch();
  sqrt_scalar_kernel<<<1, 1, 0, s>>>(x);
  return cudaGetLastError();
}

cudaError_t colsdot_launch(const double2* v, long long ldv, int n, int ncols, const double2* r,
                           double2* out, const int* done, cudaStream_t s) {
  if (ncols <= 0) return cudaSuccess;
  note_launch();
  colsdot_kernel<<<ncols, 256, 0, s>>>(v, ldv, n, r, out, done);
  return cudaGetLastError();
}

cudaError_t sub_vcoef_launch(const double2* v, long long ldv, int n, int ncols,
                             const double2* coef, double2* r, const int* done, cudaStream_t s) {
  if (ncols <= 0) return cudaSuccess;
  note_launch();
  sub_vcoef_kernel<<<(n + 127) / 128, 128, 0, s>>>(v, ldv, n, ncols, coef, r, done);
  return cudaGetLastError();
}

cudaError_t lanczos_residual_launch(const double2* u, const double2* q, const double2* qprev,
                                    const double* alpha_i, const double* beta_prev, double2* r,
                                    int n, const int* done, cudaStream_t s) {
  note_launch();
  lanczos_residual_kernel<<<(n + 255) / 256, 256, 0, s>>>(u, q, qprev, alpha_i, beta_prev, r, n,
                                                          done);
  return cudaGetLastError();
}

cudaError_t lanczos_advance_launch(const double2* r, const double* beta, double2* qnext,
                                   double* betas_i, LanczosState* st, int i, int k, int n,
                                   cudaStream_t s) {
  note_launch();
  lanczos_advance_kernel<<<(n + 255) / 256, 256, 0, s>>>(r, beta, qnext, betas_i, st, i, k, n);
  return cudaGetLastError();
}

cudaError_t colnorm_residual_launch(const double2* hp, long long ldhp, const double2* p,
                                    long long ldp, const double* lambda, int n, int w,
                                    double* res, cudaStream_t s, bool squared) {
  if (w <= 0) return cudaSuccess;
  note_launch();
  colnorm_residual_kernel<<<w, 256, 0, s>>>(hp, ldhp, p, ldp, lambda, n, res, squared ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t colnorm_launch(const double2* x, long long ldx, int n, int w, double* res,
                           cudaStream_t s) {
  return colnorm_residual_launch(x, ldx, nullptr, 0, nullptr, n, w, res, s);
}

cudaError_t symmetrize_launch(double2* a, long long lda, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int nb = (n + TS - 1) / TS;
  note_launch();
  symmetrize_kernel<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(a, lda, n);
  return cudaGetLastError();
}

cudaError_t herm_defect_launch(const double2* a, long long lda, int n, double* out,
                               cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(double), s);
  if (e != cudaSuccess || n <= 0) return e;
  const int nb = (n + TS - 1) / TS;
  note_launch();
  herm_defect_kernel<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(
      a, lda, n, reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

cudaError_t conj_transpose_launch(const double2* src, long long lds, double2* dst, long long ldd, int n,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int nb = (n + TS - 1) / TS;
  note_launch();
  conj_transpose_kernel<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(src, lds, dst, ldd, n);
  return cudaGetLastError();
}

cudaError_t conj_inplace_launch(double2* a, long long lda, int m, int n, cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  note_launch();
  conj_inplace_kernel<<<grid_for((long long)m * n, 256), 256, 0, s>>>(a, lda, m, n);
  return cudaGetLastError();
}

cudaError_t zero_upper_launch(double2* a, long long lda, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  note_launch();
  zero_upper_kernel<<<grid_for((long long)n * n, 256), 256, 0, s>>>(a, lda, n);
  return cudaGetLastError();
}

cudaError_t phase_fix_launch(double2* q, long long ldq, int m, int n, const double2* rdiag,
                             cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  note_launch();
  phase_fix_kernel<<<grid_for((long long)m * n, 256), 256, 0, s>>>(q, ldq, m, n, rdiag);
  return cudaGetLastError();
}

cudaError_t extract_diag_launch(const double2* a, long long lda, int n, double2* diag,
                                cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  note_launch();
  extract_diag_kernel<<<(n + 255) / 256, 256, 0, s>>>(a, lda, n, diag);
  return cudaGetLastError();
}

cudaError_t div_scalar_launch(const double2* x, const double* d, double2* y, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  note_launch();
  div_scalar_kernel<<<(n + 255) / 256, 256, 0, s>>>(x, d, y, n);
  return cudaGetLastError();
}

cudaError_t add_diag_shift_launch(double2* a, long long lda, int n, const double* fro, double coef,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  note_launch();
  add_diag_shift_kernel<<<(n + 255) / 256, 256, 0, s>>>(a, lda, n, fro, coef);
  return cudaGetLastError();
}

cudaError_t diag_accumulate_launch(const double2* r, long long ldr, int n, double* acc, bool first,
                                   cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  note_launch();
  diag_accumulate_kernel<<<(n + 255) / 256, 256, 0, s>>>(r, ldr, n, acc, first ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t cheb_first_step_launch(const double2* hy, long long ldhy, const double2* y0, long long ldy,
                                   double2* out, long long ldo, int n, int w, double alpha, double c,
                                   cudaStream_t s) {
  if (n <= 0 || w <= 0) return cudaSuccess;
  note_launch();
  cheb_first_step_kernel<<<grid_for((long long)n * w, 256), 256, 0, s>>>(hy, ldhy, y0, ldy, out, ldo,
                                                                         n, w, alpha, c);
  return cudaGetLastError();
}

cudaError_t near_identity_update_launch(double2* g, long long ldg, int n, double* acc, double* last,
                                        double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  note_launch();
  near_identity_update_kernel<<<1, kNiThreads, 0, s>>>(g, ldg, n, acc, last, out);
  return cudaGetLastError();
}

cudaError_t copy_cols_launch(const double2* x, long long ldx, double2* y, long long ldy, int m,
                             int n, cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  note_launch();
  copy_cols_kernel<<<grid_for((long long)m * n, 256), 256, 0, s>>>(x, ldx, y, ldy, m, n);
  return cudaGetLastError();
}

}  // namespace chfsi
