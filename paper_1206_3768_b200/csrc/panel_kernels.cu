// Panel kernels of the Cholesky-QR2 orthonormalisation (reference
// spectral_chain/chfsi.py:242-261 -> linalg.py:152-178; here Cholesky-QR2,
// chfsi_abi.cu qr_cholqr) for the panel widths of the ChFSI loop
// (w <= kPanelMaxW): the tall-skinny right-hand operations that cuBLAS runs
// as latency-bound kernel chains at these shapes (2048 x 160: ZTRSM 47-73 us;
// near-identity update + ZGEMM + copy-back ~45 us) as ONE row-parallel
// kernel each.
//
//   post_potrf  diag(L) bookkeeping of the acceptance test and the inverses
//               of L's 16x16 diagonal blocks (one warp per block)
//   right<0>    Y <- Y L^-H   (block forward substitution over 16-column
//               blocks; the diagonal solves are products with the inverted
//               blocks, so nothing in the kernel is sequential per column)
//   right<1>    Y <- Y M,  M = I - tri(G2 - I) formed on the fly from the
//               second pass's Gram matrix G2 (linearised second pass), plus
//               the pass's statistics (max|E|, R2 diagonal)
//
// Each CTA owns 16 rows of Y, keeps them in shared memory for the whole
// operation (Y is read and written once), and streams the w x w factor
// through shared memory one 16-column block at a time (L2-resident: 410 KB at
// w = 160). Fixed summation order: bitwise reproducible.
#include "chfsi_internal.h"
#include "common.cuh"

namespace chfsi {

namespace {

constexpr int PK_THREADS = 256;

__device__ __forceinline__ void cmac(double2& acc, const double2 a, const double2 b) {  // acc += a b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ void cmac_conj(double2& acc, const double2 a, const double2 b) {  // acc += a conj(b)
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
}

// One warp per 16x16 diagonal block of the lower Cholesky factor L (g, ld
// ldg): acc[i] = (first ? 1 : acc[i]) * L_ii, last[i] = L_ii (when given),
// linv[b][j*16 + i] = (L_bb^-1)[i][j] (lower; blocks past n padded with the
// identity), *eps = 0 (the linearised pass accumulates its maximum there).
__global__ void __launch_bounds__(32) panel_post_potrf_kernel(const double2* g, long long ldg, int n,
                                                              double* acc, int first, double* last,
                                                              double2* linv, double* eps) {
  __shared__ double2 Lb[16][17];
  __shared__ double2 Xb[16][17];
  const int b = blockIdx.x, lane = threadIdx.x, b16 = b * 16;
  for (int idx = lane; idx < 256; idx += 32) {
    const int c = idx >> 4, r = idx & 15;
    const int gi = b16 + r, gj = b16 + c;
    double2 v = make_double2(r == c ? 1.0 : 0.0, 0.0);
    if (r >= c && gi < n) v = g[(long long)gj * ldg + gi];
    Lb[r][c] = v;
    Xb[r][c] = make_double2(0.0, 0.0);
  }
  __syncwarp();
  if (lane < 16) {
    const int i = b16 + lane;
    if (i < n) {
      const double d = Lb[lane][lane].x;
      acc[i] = (first ? 1.0 : acc[i]) * d;
      if (last) last[i] = d;
    }
    // column j = lane of X = L_bb^-1 by forward substitution (real diagonal);
    // the column stays in registers (fully unrolled: entries above j are zero)
    const int j = lane;
    double2 x[16];
#pragma unroll
    for (int i2 = 0; i2 < 16; ++i2) {
      double2 s = make_double2(i2 == j ? -1.0 : 0.0, 0.0);  // -(e_j)_i + sum_{k < i} L_ik x_k
#pragma unroll
      for (int k = 0; k < i2; ++k) cmac(s, Lb[i2][k], x[k]);
      const double inv = 1.0 / Lb[i2][i2].x;
      x[i2] = i2 < j ? make_double2(0.0, 0.0) : make_double2(-s.x * inv, -s.y * inv);
    }
#pragma unroll
    for (int i2 = 0; i2 < 16; ++i2) Xb[i2][j] = x[i2];
  }
  __syncwarp();
  for (int idx = lane; idx < 256; idx += 32) {
    const int j = idx >> 4, i = idx & 15;
    linv[(long long)b * 256 + idx] = Xb[i][j];
  }
  if (b == 0 && lane == 0 && eps) *eps = 0.0;
}

// shared memory: the CTA's rows [np][16], two factor-block buffers [np][17]
// (cp.async double buffering), the k-parity hand-over and T tiles, two
// inverted-diagonal-block buffers
__host__ __device__ constexpr size_t panel_smem_bytes(int np) {
  return ((size_t)np * 16 + 2 * (size_t)np * 17 + 4 * 256) * sizeof(double2);
}

// MODE 0: Y <- Y L^-H (L lower in g, inverted diagonal blocks in linv).
// MODE 1: Y <- Y M, M = I - tri(E), E = G2 - I (G2 upper in g); statistics:
//         *eps = max(*eps, max |Re/Im E_ij|, i <= j) (NaN propagates),
//         acc[j] *= 1 + E_jj / 2, last[j] = 1 + E_jj / 2.
// 256 threads: r = tid & 15 (row), cg = (tid >> 4) & 7 (columns cg, cg + 8 of
// the current 16-column block), kh = tid >> 7 (even / odd k of the
// off-diagonal products; the halves are added in fixed order). The factor
// block of step b + 1 streams into the other buffer (cp.async) while step b
// computes.
template <int MODE>
__global__ void __launch_bounds__(PK_THREADS) panel_right_kernel(double2* y, long long ld, int m, int n,
                                                                 const double2* g, long long ldg,
                                                                 const double2* linv, double* acc,
                                                                 double* last, double* eps) {
  extern __shared__ double2 psm[];
  const int t16 = (n + 15) >> 4, np = t16 * 16;
  double2* Xs = psm;                        // [np][16]: column c, row r at c * 16 + r
  double2* Fbuf = Xs + (size_t)np * 16;     // 2 x [np][17]: factor block, k * 17 + c
  double2* Ps = Fbuf + 2 * (size_t)np * 17; // [16][16]: odd-k partial sums, c * 16 + r
  double2* Ts = Ps + 256;                   // [16][16]: c * 16 + r
  double2* Lbuf = Ts + 256;                 // 2 x [16][16]: k * 16 + c = (L_bb^-1)[c][k]
  const int tid = threadIdx.x, r = tid & 15, cg = (tid >> 4) & 7, kh = tid >> 7;
  const int r0 = blockIdx.x * 16;
  const double2 zero = make_double2(0.0, 0.0);
  // factor block b into buffer `buf` (asynchronous; zero fill outside the matrix)
  auto stage = [&](int b, int buf) {
    double2* Fs = Fbuf + (size_t)buf * np * 17;
    const int b16 = b * 16;
    if (MODE == 0) {  // Fs[k][c] = L[b16 + c][k], k < b16 (c contiguous in memory)
      for (int idx = tid; idx < b16 * 16; idx += PK_THREADS) {
        const int k = idx >> 4, c = idx & 15;
        const bool ok = b16 + c < n;
        cp_async16(&Fs[k * 17 + c], &g[(long long)k * ldg + (ok ? b16 + c : 0)], ok);
      }
      double2* Li = Lbuf + buf * 256;
      cp_async16(&Li[tid], &linv[(long long)b * 256 + tid], true);
    } else {  // Fs[k][c] = G2[k][b16 + c], k < b16 + 16 (k contiguous in memory)
      const int klen = b16 + 16;
      for (int idx = tid; idx < klen * 16; idx += PK_THREADS) {
        const int c = idx / klen, k = idx - c * klen, j = b16 + c;
        const bool ok = j < n && k < n;
        cp_async16(&Fs[k * 17 + c], &g[(long long)(ok ? j : 0) * ldg + (ok ? k : 0)], ok);
      }
    }
  };
  for (int idx = tid; idx < np * 16; idx += PK_THREADS) {
    const int c = idx >> 4, rr = idx & 15;
    const bool ok = c < n && r0 + rr < m;
    cp_async16(&Xs[idx], &y[ok ? (long long)c * ld + r0 + rr : 0], ok);
  }
  const int first = MODE == 0 ? 0 : t16 - 1, step = MODE == 0 ? 1 : -1;
  stage(first, 0);
  cp_async_commit();
  for (int it = 0; it < t16; ++it) {
    const int b = first + it * step, b16 = b * 16, buf = it & 1;
    const double2* Fs = Fbuf + (size_t)buf * np * 17;
    if (it + 1 < t16) stage(b + step, buf ^ 1);  // (that buffer's readers finished in step it - 1)
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();  // this step's factor block (and Xs) landed; the previous step's Xs columns are written
    // off-diagonal products over k < b16, even / odd k by thread half:
    //   MODE 0: sum_k X[r][k] conj(L[b16 + c][k]);  MODE 1: sum_k X[r][k] G2[k][b16 + c]
    // (b16 / 2 k values per thread, a multiple of 8: four independent
    // accumulator pairs, the twelve operand loads of a group issued ahead
    // of its sixteen complex MACs)
    double2 s0, s1;
    {
      double2 p0[4] = {zero, zero, zero, zero}, p1[4] = {zero, zero, zero, zero};
      for (int k = kh; k < b16; k += 8) {
        double2 x[4], f0[4], f1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[u] = Xs[(k + 2 * u) * 16 + r];
          f0[u] = Fs[(k + 2 * u) * 17 + cg];
          f1[u] = Fs[(k + 2 * u) * 17 + cg + 8];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (MODE == 0) {
            cmac_conj(p0[u], x[u], f0[u]);
            cmac_conj(p1[u], x[u], f1[u]);
          } else {
            cmac(p0[u], x[u], f0[u]);
            cmac(p1[u], x[u], f1[u]);
          }
        }
      }
      s0 = make_double2((p0[0].x + p0[1].x) + (p0[2].x + p0[3].x), (p0[0].y + p0[1].y) + (p0[2].y + p0[3].y));
      s1 = make_double2((p1[0].x + p1[1].x) + (p1[2].x + p1[3].x), (p1[0].y + p1[1].y) + (p1[2].y + p1[3].y));
    }
    if (kh) {
      Ps[cg * 16 + r] = s0;
      Ps[(cg + 8) * 16 + r] = s1;
    }
    __syncthreads();
    if (MODE == 0) {
      if (!kh) {  // T = Y_b - (even + odd)
        const double2 p0 = Ps[cg * 16 + r], p1 = Ps[(cg + 8) * 16 + r];
        const double2 a0 = Xs[(b16 + cg) * 16 + r], a1 = Xs[(b16 + cg + 8) * 16 + r];
        Ts[cg * 16 + r] = make_double2(a0.x - (s0.x + p0.x), a0.y - (s0.y + p0.y));
        Ts[(cg + 8) * 16 + r] = make_double2(a1.x - (s1.x + p1.x), a1.y - (s1.y + p1.y));
      }
      __syncthreads();
      // X_b = T L_bb^-H: X_b[r][c] = sum_{k <= c} T[r][k] conj((L_bb^-1)[c][k]);
      // thread half kh takes column cg + 8 kh
      const double2* Li = Lbuf + buf * 256;
      const int c = cg + 8 * kh;
      double2 o = zero;
      for (int kk = 0; kk <= c; ++kk) cmac_conj(o, Ts[kk * 16 + r], Li[kk * 16 + c]);
      Xs[(b16 + c) * 16 + r] = o;
    } else {
      // out[r][c] = -(even + odd) - sum_{k' < c} X[r][b16 + k'] G2[b16 + k'][j] + X[r][j] (1 - E_jj / 2);
      // thread half kh takes column cg + 8 kh (reads the block's own input columns)
      const int c = cg + 8 * kh;
      if (!kh) {  // even-k sums through Ts (the odd ones are in Ps)
        Ts[cg * 16 + r] = s0;
        Ts[(cg + 8) * 16 + r] = s1;
      }
      __syncthreads();
      const double2 ev = Ts[c * 16 + r], od = Ps[c * 16 + r];
      double2 d = zero;
      for (int kk = 0; kk < c; ++kk) cmac(d, Xs[(b16 + kk) * 16 + r], Fs[(b16 + kk) * 17 + c]);
      const double2 xj = Xs[(b16 + c) * 16 + r];
      const double mjj = 1.0 - 0.5 * (Fs[(b16 + c) * 17 + c].x - 1.0);
      const double2 o = make_double2(xj.x * mjj - ((ev.x + od.x) + d.x), xj.y * mjj - ((ev.y + od.y) + d.y));
      __syncthreads();  // every thread has read the block's own input columns
      Xs[(b16 + c) * 16 + r] = o;
    }
    __syncthreads();  // this step's buffers are free for the prefetch after next; its Xs columns are final
  }
  for (int idx = tid; idx < np * 16; idx += PK_THREADS) {
    const int c = idx >> 4, rr = idx & 15;
    if (c < n && r0 + rr < m) y[(long long)c * ld + r0 + rr] = Xs[idx];
  }
  if (MODE == 1) {
    // statistics of E = G2 - I, column j by CTA j % grid (max is exact: order-free)
    __shared__ double red[PK_THREADS / 32];
    for (int j = blockIdx.x; j < n; j += gridDim.x) {
      double emax = 0.0;
      for (int i = tid; i <= j; i += PK_THREADS) {
        const double2 e = __ldcg(&g[(long long)j * ldg + i]);
        double a = fabs(i == j ? e.x - 1.0 : e.x);
        const double bq = fabs(e.y);
        a = (bq > a || bq != bq) ? bq : a;
        emax = (a > emax || a != a) ? a : emax;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_down_sync(0xffffffffu, emax, o);
        emax = (t > emax || t != t) ? t : emax;
      }
      __syncthreads();
      if ((tid & 31) == 0) red[tid >> 5] = emax;
      __syncthreads();
      if (tid == 0) {
        double mx = 0.0;
        for (int w = 0; w < PK_THREADS / 32; ++w) mx = (red[w] > mx || red[w] != red[w]) ? red[w] : mx;
        // non-negative doubles and NaNs order like their bit patterns
        atomicMax(reinterpret_cast<unsigned long long*>(eps),
                  (unsigned long long)__double_as_longlong(fabs(mx)));
        const double d = __ldcg(&g[(long long)j * ldg + j].x) - 1.0;
        const double r2 = 1.0 + 0.5 * d;
        acc[j] *= r2;
        last[j] = r2;
      }
    }
  }
}

template <int MODE>
cudaError_t panel_right_launch(double2* y, long long ld, int m, int n, const double2* g, long long ldg,
                               const double2* linv, double* acc, double* last, double* eps,
                               cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  if (n > kPanelMaxW) return cudaErrorInvalidValue;
  static const cudaError_t attr = cudaFuncSetAttribute(
      reinterpret_cast<const void*>(panel_right_kernel<MODE>),
      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)panel_smem_bytes(kPanelMaxW));
  if (attr != cudaSuccess) return attr;
  const int np = ((n + 15) / 16) * 16;
  note_launch();
  panel_right_kernel<MODE><<<(m + 15) / 16, PK_THREADS, panel_smem_bytes(np), s>>>(y, ld, m, n, g, ldg, linv,
                                                                                 acc, last, eps);
  return cudaGetLastError();
}

}  // namespace

size_t panel_linv_bytes() { return (size_t)(kPanelMaxW / 16) * 256 * sizeof(double2); }

cudaError_t panel_post_potrf_launch(const double2* g, long long ldg, int n, double* acc, bool first,
                                    double* last, double2* linv, double* eps, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > kPanelMaxW) return cudaErrorInvalidValue;
  note_launch();
  panel_post_potrf_kernel<<<(n + 15) / 16, 32, 0, s>>>(g, ldg, n, acc, first ? 1 : 0, last, linv, eps);
  return cudaGetLastError();
}

cudaError_t panel_trsm_lh_launch(double2* y, long long ld, int m, int n, const double2* l, long long ldl,
                                 const double2* linv, cudaStream_t s) {
  return panel_right_launch<0>(y, ld, m, n, l, ldl, linv, nullptr, nullptr, nullptr, s);
}

cudaError_t panel_apply_near_identity_launch(double2* y, long long ld, int m, int n, const double2* g2,
                                             long long ldg, double* acc, double* last, double* eps,
                                             cudaStream_t s) {
  return panel_right_launch<1>(y, ld, m, n, g2, ldg, nullptr, acc, last, eps, s);
}

}  // namespace chfsi
