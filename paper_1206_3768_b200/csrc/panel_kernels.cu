// Panel kernels of the Cholesky-QR2 orthonormalisation (reference
// spectral_chain/chfsi.py:242-261 -> linalg.py:152-178; here Cholesky-QR2,
// chfsi_abi.cu qr_cholqr) for the panel widths of the ChFSI loop
// (w <= kPanelMaxW): the tall-skinny right-hand operations that cuBLAS runs
// as latency-bound kernel chains at these shapes (2048 x 160: ZTRSM 47-73 us;
// near-identity update + ZGEMM + copy-back ~45 us) as ONE row-parallel
// kernel each.
//
//   post_potrf  diag(L) bookkeeping of the acceptance test and the inverses
//               of L's 16x16 diagonal blocks (one CTA per block)
//   right<0>    Y <- Y L^-H   (block forward substitution over 16-column
//               blocks; the diagonal solves are products with the inverted
//               blocks, so nothing in the kernel is sequential per column)
//   right<1>    Y <- Y M,  M = I - tri(G2 - I) formed on the fly from the
//               second pass's Gram matrix G2 (linearised second pass), plus
//               the pass's statistics (max|E|, R2 diagonal)
//
// (Measured and rejected: the w x w Cholesky itself as ONE hand-written CTA —
// left-looking 16-column blocks, DMMA updates from staged L rows,
// right-looking block-column factorisation in shared memory, fused with
// post_potrf's work. Correct against every QR test, but one SM's worth of
// FP64 plus ~10 serial block steps took 174 us at w = 160 against cuSOLVER
// potrf's 71 us (level at w <= 48); C2 ortho 31 -> 35 ms. potrf stays.)
//
// Each CTA owns 16 rows of Y, keeps them in shared memory for the whole
// operation (Y is read and written once), and streams the w x w factor
// through shared memory one 16-column block at a time (L2-resident: 410 KB at
// w = 160). Fixed summation order: bitwise reproducible.
#include "chfsi_internal.h"
#include "common.cuh"

namespace chfsi {

namespace {

constexpr int PK_THREADS = 512;

__device__ __forceinline__ void cmac(double2& acc, const double2 a, const double2 b) {  // acc += a b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// One CTA per 16x16 diagonal block of the lower Cholesky factor L (g, ld
// ldg): acc[i] = (first ? 1 : acc[i]) * L_ii, last[i] = L_ii (when given),
// linv[b][j*16 + i] = (L_bb^-1)[i][j] (lower; blocks past n padded with the
// identity), *eps = 0 (the linearised pass accumulates its maximum there).
__global__ void __launch_bounds__(256) panel_post_potrf_kernel(const double2* g, long long ldg, int n,
                                                               double* acc, int first, double* last,
                                                               double2* linv, double* eps) {
  __shared__ double2 Lb[16][17];
  __shared__ double2 Xb[16][17];
  const int b = blockIdx.x, tid = threadIdx.x, b16 = b * 16;
  {  // one tile element per thread (one L2 latency for the whole tile)
    const int c = tid >> 4, r = tid & 15;
    const int gi = b16 + r, gj = b16 + c;
    double2 v = make_double2(r == c ? 1.0 : 0.0, 0.0);
    if (r >= c && gi < n) v = g[(long long)gj * ldg + gi];
    Lb[r][c] = v;
  }
  __syncthreads();
  if (tid < 16) {
    const int i = b16 + tid;
    if (i < n) {
      const double d = Lb[tid][tid].x;
      acc[i] = (first ? 1.0 : acc[i]) * d;
      if (last) last[i] = d;
    }
    // column j = tid of X = L_bb^-1 by forward substitution (real diagonal);
    // the column stays in registers (fully unrolled: entries above j are zero)
    const int j = tid;
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
  __syncthreads();
  linv[(long long)b * 256 + tid] = Xb[tid & 15][tid >> 4];
  if (b == 0 && tid == 0 && eps) *eps = 0.0;
}

// shared memory (complex elements): the CTA's rows [np][XS], two factor-block
// buffers [np][FS] (cp.async double buffering), the off-diagonal partial
// tiles [4 k-quarters][4 blocks][32 lanes][2], T [16][XS], two
// inverted-diagonal-block buffers [16][FS]. Row strides of 18 elements
// (288 B) keep the 16-byte DMMA fragment loads bank-conflict free.
constexpr int XS = 18, FS = 18;
__host__ __device__ constexpr size_t panel_smem_bytes(int np) {
  return ((size_t)np * XS + 2 * ((size_t)np * FS + 64) + 1024 + 16 * XS + 2 * 16 * FS) * sizeof(double2);
}

// complex 8x8x4 block on DMMA: (cr, ci) += a b (CONJ_B: a conj(b)), four real products
template <bool CONJ_B>
__device__ __forceinline__ void zmma884(double (&cr)[2], double (&ci)[2], const double2 a, const double2 b) {
  dmma884(cr, a.x, b.x);
  dmma884(cr, CONJ_B ? a.y : -a.y, b.y);
  dmma884(ci, a.y, b.x);
  dmma884(ci, CONJ_B ? -a.x : a.x, b.y);
}

// MODE 0: Y <- Y L^-H (L lower in g, inverted diagonal blocks in linv).
// MODE 1: Y <- Y M, M = I - tri(E), E = G2 - I (G2 upper in g); statistics:
//         *eps = max(*eps, max |Re/Im E_ij|, i <= j) (NaN propagates),
//         acc[j] *= 1 + E_jj / 2, last[j] = 1 + E_jj / 2.
// 16 warps. Per 16-column block b the 16 x 16 output tile is four 8x8 DMMA
// blocks (blk = row half + 2 column half); warp w accumulates block w & 3
// over the k4 steps congruent to w >> 2 mod 4 of the off-diagonal product
// (fragments straight from shared memory: two 16-byte loads per four
// DMMA.8x8x4 — the FFMA-style version of this kernel was bound by
// shared-memory wavefronts at 29 % of the FP64 pipe); the four k-quarters
// are added in fixed order, and warps 0-3 finish the block (diagonal
// product, also on DMMA). The factor block of step b + 1 streams into the
// other buffer (cp.async) while step b computes.
template <int MODE>
__global__ void __launch_bounds__(PK_THREADS) panel_right_kernel(double2* y, long long ld, int m, int n,
                                                                 const double2* g, long long ldg,
                                                                 const double2* linv, double* acc,
                                                                 double* last, double* eps) {
  extern __shared__ double2 psm[];
  const int t16 = (n + 15) >> 4, np = t16 * 16;
  double2* Xs = psm;                        // [np][XS]: column c, row r at c * XS + r
  double2* Fbuf = Xs + (size_t)np * XS;     // 2 x [np][FS]: factor block, k * FS + c
  double2* Ps = Fbuf + 2 * ((size_t)np * FS + 64);  // [4][4][32][2]: partial C fragments
  double2* Ts = Ps + 1024;                  // [16][XS]: T, column kk, row r at kk * XS + r
  double2* Lbuf = Ts + 16 * XS;             // 2 x [16][FS]: k * FS + c = (L_bb^-1)[c][k]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, gq = lane >> 2, t = lane & 3;
  const int blk = w & 3, kq = w >> 2, rb = blk & 1, cb = blk >> 1;
  const int r0 = blockIdx.x * 16;
  const int ks = np + 4;  // MODE 1: k-stride of the column-major factor block
  const double2 zero = make_double2(0.0, 0.0);
  // factor block b into buffer `buf` (asynchronous; zero fill outside the matrix)
  auto stage = [&](int b, int buf) {
    double2* Fs = Fbuf + (size_t)buf * (np * FS + 64);
    const int b16 = b * 16;
    if (MODE == 0) {  // Fs[k][c] = L[b16 + c][k], k < b16 (c contiguous in memory)
      for (int idx = tid; idx < b16 * 16; idx += PK_THREADS) {
        const int k = idx >> 4, c = idx & 15;
        const bool ok = b16 + c < n;
        cp_async16(&Fs[k * FS + c], &g[(long long)k * ldg + (ok ? b16 + c : 0)], ok);
      }
      double2* Li = Lbuf + buf * 16 * FS;
      if (tid < 256) cp_async16(&Li[(tid >> 4) * FS + (tid & 15)], &linv[(long long)b * 256 + tid], true);
    } else {  // G2[k][b16 + c], k < b16 + 16, stored column-major (c * ks + k: k contiguous in global
              // and shared memory, conflict-free copies; ks = 4 mod 8 keeps the fragment loads so)
      const int klen = b16 + 16;
      for (int idx = tid; idx < klen * 16; idx += PK_THREADS) {
        const int c = idx / klen, k = idx - c * klen, j = b16 + c;
        const bool ok = j < n && k < n;
        cp_async16(&Fs[c * ks + k], &g[(long long)(ok ? j : 0) * ldg + (ok ? k : 0)], ok);
      }
    }
  };
  for (int idx = tid; idx < np * 16; idx += PK_THREADS) {
    const int c = idx >> 4, rr = idx & 15;
    const bool ok = c < n && r0 + rr < m;
    cp_async16(&Xs[c * XS + rr], &y[ok ? (long long)c * ld + r0 + rr : 0], ok);
  }
  const int first = MODE == 0 ? 0 : t16 - 1, step = MODE == 0 ? 1 : -1;
  stage(first, 0);
  cp_async_commit();
  for (int it = 0; it < t16; ++it) {
    const int b = first + it * step, b16 = b * 16, buf = it & 1;
    const double2* Fs = Fbuf + (size_t)buf * (np * FS + 64);
    if (it + 1 < t16) stage(b + step, buf ^ 1);  // (that buffer's readers finished in step it - 1)
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();  // this step's factor block (and Xs) landed; the previous step's Xs columns are written
    // off-diagonal product over k < b16:
    //   MODE 0: sum_k X[r][k] conj(L[b16 + c][k]);  MODE 1: sum_k X[r][k] G2[k][b16 + c]
    {
      double cr0[2] = {0.0, 0.0}, ci0[2] = {0.0, 0.0}, cr1[2] = {0.0, 0.0}, ci1[2] = {0.0, 0.0};
      const double2* xa = Xs + t * XS + rb * 8 + gq;
      const double2* fb = MODE == 0 ? Fs + t * FS + cb * 8 + gq : Fs + (cb * 8 + gq) * ks + t;
      const int fstep = MODE == 0 ? 4 * FS : 4;  // one k4 step in the factor block
      const int nk4 = b16 >> 2;
      int k4 = kq;
      for (; k4 + 4 < nk4; k4 += 8) {  // two steps per trip on independent accumulators
        const double2 a0 = xa[4 * k4 * XS], f0 = fb[k4 * fstep];
        const double2 a1 = xa[4 * (k4 + 4) * XS], f1 = fb[(k4 + 4) * fstep];
        zmma884<MODE == 0>(cr0, ci0, a0, f0);
        zmma884<MODE == 0>(cr1, ci1, a1, f1);
      }
      if (k4 < nk4) zmma884<MODE == 0>(cr0, ci0, xa[4 * k4 * XS], fb[k4 * fstep]);
      double2* pp = Ps + ((kq * 4 + blk) * 32 + lane) * 2;
      pp[0] = make_double2(cr0[0] + cr1[0], ci0[0] + ci1[0]);
      pp[1] = make_double2(cr0[1] + cr1[1], ci0[1] + ci1[1]);
    }
    __syncthreads();
    if (MODE == 0) {
      if (tid < 128) {  // T = Y_b - (k-quarters 0..3 in fixed order); thread = (block, lane) of the
                        // C fragments, both of its elements: consecutive lanes read consecutive 32 bytes
        const int fb = tid >> 5, fl = tid & 31;
        const double2* pp = Ps + (fb * 32 + fl) * 2;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = (fb & 1) * 8 + (fl >> 2), c = (fb >> 1) * 8 + 2 * (fl & 3) + e;
          const double2 p0 = pp[e], p1 = pp[256 + e], p2 = pp[512 + e], p3 = pp[768 + e];
          const double2 yv = Xs[(b16 + c) * XS + r];
          Ts[c * XS + r] =
              make_double2(yv.x - ((p0.x + p1.x) + (p2.x + p3.x)), yv.y - ((p0.y + p1.y) + (p2.y + p3.y)));
        }
      }
      __syncthreads();
      if (w < 4) {  // X_b = T L_bb^-H: X_b[r][c] = sum_k T[r][k] conj((L_bb^-1)[c][k]) (zero for k > c)
        const double2* Li = Lbuf + buf * 16 * FS;
        double cr[4][2] = {}, ci[4][2] = {};  // one accumulator pair per k4 step: no DMMA chain
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4)
          zmma884<true>(cr[k4], ci[k4], Ts[(4 * k4 + t) * XS + rb * 8 + gq], Li[(4 * k4 + t) * FS + cb * 8 + gq]);
#pragma unroll
        for (int e = 0; e < 2; ++e)
          Xs[(b16 + cb * 8 + 2 * t + e) * XS + rb * 8 + gq] =
              make_double2((cr[0][e] + cr[1][e]) + (cr[2][e] + cr[3][e]), (ci[0][e] + ci[1][e]) + (ci[2][e] + ci[3][e]));
      }
    } else {
      // out[r][c] = X[r][j] (1 - E_jj / 2) - sum - sum_{k' < c} X[r][b16 + k'] G2[b16 + k'][j]
      // (the block's own input columns are read before any of them is overwritten)
      double2 o[2] = {zero, zero};
      if (w < 4) {
        double cr4[4][2] = {}, ci4[4][2] = {};  // one accumulator pair per k4 step: no DMMA chain
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int kk = 4 * k4 + t, cc = cb * 8 + gq;
          const double2 f = Fs[cc * ks + b16 + kk];
          zmma884<false>(cr4[k4], ci4[k4], Xs[(b16 + kk) * XS + rb * 8 + gq], kk < cc ? f : zero);
        }
        const double cr[2] = {(cr4[0][0] + cr4[1][0]) + (cr4[2][0] + cr4[3][0]),
                              (cr4[0][1] + cr4[1][1]) + (cr4[2][1] + cr4[3][1])};
        const double ci[2] = {(ci4[0][0] + ci4[1][0]) + (ci4[2][0] + ci4[3][0]),
                              (ci4[0][1] + ci4[1][1]) + (ci4[2][1] + ci4[3][1])};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = rb * 8 + gq, c = cb * 8 + 2 * t + e;
          const double2* pp = Ps + (blk * 32 + lane) * 2 + e;
          const double2 p0 = pp[0], p1 = pp[256], p2 = pp[512], p3 = pp[768];
          const double2 xj = Xs[(b16 + c) * XS + r];
          const double mjj = 1.0 - 0.5 * (Fs[c * ks + b16 + c].x - 1.0);
          o[e] = make_double2(xj.x * mjj - (((p0.x + p1.x) + (p2.x + p3.x)) + cr[e]),
                              xj.y * mjj - (((p0.y + p1.y) + (p2.y + p3.y)) + ci[e]));
        }
      }
      __syncthreads();
      if (w < 4) {
#pragma unroll
        for (int e = 0; e < 2; ++e) Xs[(b16 + cb * 8 + 2 * t + e) * XS + rb * 8 + gq] = o[e];
      }
    }
    __syncthreads();  // this step's buffers are free for the prefetch after next; its Xs columns are final
  }
  for (int idx = tid; idx < np * 16; idx += PK_THREADS) {
    const int c = idx >> 4, rr = idx & 15;
    if (c < n && r0 + rr < m) y[(long long)c * ld + r0 + rr] = Xs[c * XS + rr];
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
        const double tt = __shfl_down_sync(0xffffffffu, emax, o);
        emax = (tt > emax || tt != tt) ? tt : emax;
      }
      __syncthreads();
      if ((tid & 31) == 0) red[tid >> 5] = emax;
      __syncthreads();
      if (tid == 0) {
        double mx = 0.0;
        for (int q = 0; q < PK_THREADS / 32; ++q) mx = (red[q] > mx || red[q] != red[q]) ? red[q] : mx;
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
  panel_post_potrf_kernel<<<(n + 15) / 16, 256, 0, s>>>(g, ldg, n, acc, first ? 1 : 0, last, linv, eps);
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
