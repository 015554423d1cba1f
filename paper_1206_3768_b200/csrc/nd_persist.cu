// The near-diagonal Rayleigh-Ritz eigensolver (nd_eig.cu's algorithm) as ONE
// cooperative persistent kernel, for the panel widths of the ChFSI loop
// (w <= kNdPersistMaxN; reference chfsi.py:347 -> linalg.py:181-206).
//
// Per step: X = I + S (S_ij = G_ij / (d_j - d_i)), W <- W X, Newton-Schulz
// polar steps W <- 1.5 W - 0.5 W (W^H W), X = G0 W, G = W^H X — every w x w
// product on DMMA.8x8x4 tensor cores (one CTA per 16x16 complex output tile,
// operand panels staged in shared memory, fixed summation order:
// deterministic), the elementwise pieces and the regime /
// convergence decisions in the same kernel between grid-wide barriers. The
// library version issues ~10 kernels and one host round trip per step
// (~120 us per step at w = 160 on a B200); here the host waits once, for
// the final status. Same decisions as heev_near_diag (chfsi_abi.cu): bail
// when max|G_ij|/|d_j - d_i| > bail or after kMaxSteps, converge when
// max|G_ij| <= tol * max(1, max|G_ii|) with the last Newton-Schulz input
// unitary to 1e-8; on failure A is untouched and the caller runs zheevd.
#include <cooperative_groups.h>

#include "chfsi_internal.h"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace chfsi {

namespace {

constexpr int ND_THREADS = 256;
constexpr int ND_WARPS = ND_THREADS / 32;
constexpr int kNdMaxSteps = 6;

struct NdParams {
  const double2* ain;  // G (Hermitian, column-major, ld lda)
  long long lda;
  double2* aout;       // sorted eigenvectors on success (may alias ain; ld lda)
  double* w;           // sorted eigenvalues on success
  int n;
  double2 *G0, *G, *X, *T, *W, *W2;  // n x n scratch, ld n
  double* part;        // [grid][4]: rmax, emax, dmax, NS defect partials
  int* perm;           // n
  double* status;      // [4]: done (1/0), steps, last rmax, last emax
  double tol, bail;
};

__device__ __forceinline__ double pmax(double a, double b) { return (b > a || isnan(b)) ? b : a; }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = pmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// block max of 4 values -> part[blockIdx.x * 4 + j] (thread 0 writes; j < nv)
__device__ void block_max_publish(double (&v)[4], int nv, int first, double* part, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = 0; j < nv; ++j) {
    const double r = warp_max(v[j]);
    if (lane == 0) sh[wid * 4 + j] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int j = 0; j < nv; ++j) {
      double r = 0.0;
      for (int k = 0; k < ND_WARPS; ++k) r = pmax(r, sh[k * 4 + j]);
      part[blockIdx.x * 4 + first + j] = r;
    }
  __syncthreads();
}

// max over every CTA's four partials (max is exact: every thread gets the
// same bits). One 16-byte-pair of loads per thread and a block reduction —
// the per-thread loop over all CTAs' partials that stood here before cost
// ~100 dependent-issue L2 loads per statistic and thread (~25 us per call).
__device__ void grid_max4(const double* part, double (&out)[4], double* sh) {
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (threadIdx.x < gridDim.x) {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcg(part + threadIdx.x * 4 + j);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double r = warp_max(v[j]);
    if (lane == 0) sh[wid * 4 + j] = r;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double r = 0.0;
    for (int k = 0; k < ND_WARPS; ++k) r = pmax(r, sh[k * 4 + j]);
    out[j] = r;
  }
  __syncthreads();
}

// X = I + S, S_ij = G_ij / (d_j - d_i); stats as nd_build_step_kernel
// (g has leading dimension ldg; copy != nullptr: also copy g into it, ld n —
// the first step reads the caller's matrix and keeps it as G0 in one pass)
__device__ void build_phase(const double2* g, long long ldg, int n, double2* x, double* part, double* sh,
                            double2* copy = nullptr) {
  const long long total = (long long)n * n;
  double st[4] = {0.0, 0.0, 0.0, 0.0};
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx % n);
    double2 out;
    if (i == j) {
      out = make_double2(1.0, 0.0);
      const double2 d = __ldcg(&g[(long long)i * ldg + i]);
      if (copy) copy[idx] = d;
      st[2] = pmax(st[2], fabs(d.x));
    } else {
      const double2 e = __ldcg(&g[(long long)j * ldg + i]);
      if (copy) copy[idx] = e;
      const double gap = __ldcg(&g[(long long)j * ldg + j].x) - __ldcg(&g[(long long)i * ldg + i].x);
      const double ae = hypot(e.x, e.y);
      st[1] = pmax(st[1], ae);
      if (ae == 0.0) {
        out = make_double2(0.0, 0.0);
      } else {
        const double ag = fabs(gap);
        st[0] = pmax(st[0], ag > 0.0 ? ae / ag : INFINITY);
        out = make_double2(e.x / gap, e.y / gap);
      }
    }
    x[(long long)j * n + i] = out;
  }
  if (!(st[0] <= 1e300)) st[0] = 1e300;  // inf / nan: "not near-diagonal"
  block_max_publish(st, 3, 0, part, sh);
}

enum { EPI_STORE = 0, EPI_NS = 1, EPI_HERM = 2, EPI_DEFECT = 3 };

// shared-memory panels of one 16x16 output tile: A [k][17] (row fastest,
// padded), B [16][n+1] (k fastest, padded), plus the k-half hand-over
__host__ __device__ constexpr size_t nd_smem_doubles2(int n) {
  return (size_t)n * 17 + 16 * (size_t)(n + 1) + 4 * 32 * 2;
}

// C = op(A) B for n x n column-major complex blocks (ld n), op(A) = A or A^H.
// One CTA per 16x16 complex output tile: the A row panel and the B column
// panel are staged in shared memory (coalesced 16-byte loads from L2), the
// 8 warps each take an 8x8 quarter and half of k on DMMA.8x8x4 (four real
// products per complex block), the two k halves are added in fixed order.
//   EPI_NS:     C = 1.5 Wsrc - 0.5 (A B)           (Newton-Schulz step)
//   EPI_HERM:   upper tiles only, mirrored (exactly Hermitian, real diagonal)
//   EPI_DEFECT: store + partial max |C - I| into *dmax
template <bool CONJ_A>
__device__ void gemm_phase(const double2* A, const double2* B, double2* C, int n, int epi,
                           const double2* Wsrc, double* dmax, double2* sm) {
  const int t16 = (n + 15) >> 4;
  const int ntiles = t16 * t16;
  const int ldk = n + 1;
  double2* As = sm;                 // As[k * 17 + r] = op(A)[r0 + r][k]
  double2* Bs = sm + (size_t)n * 17;  // Bs[c * ldk + k] = B[k][c0 + c]
  double2* red = Bs + 16 * (size_t)ldk;  // [4 warps][32 lanes][2] partial (cr, ci) pairs
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, wid = threadIdx.x >> 5;
  const int sub = wid & 3, kh = wid >> 2;
  const int sr = (sub & 1) * 8, sc = (sub >> 1) * 8;
  const int kmid = min(n, ((n / 2) + 3) & ~3);
  const int kb = kh ? kmid : 0, ke = kh ? n : kmid;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int ti = tile % t16, tj = tile / t16;
    if (epi == EPI_HERM && ti > tj) continue;  // (uniform over the CTA)
    const int r0 = ti * 16, c0 = tj * 16;
    __syncthreads();  // the previous tile's panel reads are done
    // Panels by cp.async (16-byte copies from L2, all in flight at once: the
    // plain load -> store loops serialised ~10 L2 latencies per panel and
    // were most of a phase's ~7 us); op(A) = A^H is conjugated in the MMA.
    {
      const int hi = threadIdx.x >> 4, lo = threadIdx.x & 15;  // 16 x 16 thread grid
      if (!CONJ_A) {  // As[k][r] = A[r0 + r][k]: r contiguous in memory
        for (int k = hi; k < n; k += 16)
          cp_async16(&As[k * 17 + lo], &A[(long long)k * n + (r0 + lo < n ? r0 + lo : 0)], r0 + lo < n);
      } else {        // As[k][r] = A[k][r0 + r] (conjugated later): k contiguous in memory
        const bool ok = r0 + hi < n;
        for (int k = lo; k < n; k += 16)
          cp_async16(&As[k * 17 + hi], &A[(long long)(ok ? r0 + hi : 0) * n + k], ok);
      }
      const bool okb = c0 + hi < n;
      for (int k = lo; k < n; k += 16)  // Bs[c][k] = B[k][c0 + c]: k contiguous in memory
        cp_async16(&Bs[hi * ldk + k], &B[(long long)(okb ? c0 + hi : 0) * n + k], okb);
      cp_async_commit();
      cp_async_wait<0>();
    }
    __syncthreads();
    // two k4 steps per trip on independent accumulator pairs (the four DMMAs
    // of a step form two dependent pairs; one pair of chains per step parity)
    double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0}, cr1[2] = {0.0, 0.0}, ci1[2] = {0.0, 0.0};
    auto frag = [&](int k, double2& a, double2& b) {
      const bool ok = k < ke;
      a = ok ? As[k * 17 + sr + g] : make_double2(0.0, 0.0);
      b = ok ? Bs[(sc + g) * ldk + k] : make_double2(0.0, 0.0);
      if (CONJ_A) a.y = -a.y;  // op(A) = A^H: the staged panel holds A
    };
    for (int k0 = kb; k0 < ke; k0 += 8) {
      double2 a0, b0, a1, b1;
      frag(k0 + t, a0, b0);
      frag(k0 + 4 + t, a1, b1);  // (past ke: zeros)
      dmma884(cr, a0.x, b0.x);
      dmma884(cr1, a1.x, b1.x);
      dmma884(ci, a0.x, b0.y);
      dmma884(ci1, a1.x, b1.y);
      dmma884(cr, -a0.y, b0.y);
      dmma884(cr1, -a1.y, b1.y);
      dmma884(ci, a0.y, b0.x);
      dmma884(ci1, a1.y, b1.x);
    }
    cr[0] += cr1[0];
    cr[1] += cr1[1];
    ci[0] += ci1[0];
    ci[1] += ci1[1];
    if (kh) {
      red[(sub * 32 + lane) * 2 + 0] = make_double2(cr[0], cr[1]);
      red[(sub * 32 + lane) * 2 + 1] = make_double2(ci[0], ci[1]);
    }
    __syncthreads();
    if (kh) continue;
    const double2 pr = red[(sub * 32 + lane) * 2 + 0], pi = red[(sub * 32 + lane) * 2 + 1];
    cr[0] += pr.x;
    cr[1] += pr.y;
    ci[0] += pi.x;
    ci[1] += pi.y;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int row = r0 + sr + g, col = c0 + sc + 2 * t + e;
      if (row >= n || col >= n) continue;
      double2 v = make_double2(cr[e], ci[e]);
      if (epi == EPI_NS) {
        const double2 s = __ldcg(&Wsrc[(long long)col * n + row]);
        v = make_double2(1.5 * s.x - 0.5 * v.x, 1.5 * s.y - 0.5 * v.y);
      }
      if (epi == EPI_HERM) {
        if (ti == tj && row > col) continue;  // the diagonal tile's upper half is mirrored
        if (row == col) v.y = 0.0;
        C[(long long)col * n + row] = v;
        C[(long long)row * n + col] = make_double2(v.x, -v.y);
        continue;
      }
      if (epi == EPI_DEFECT) *dmax = pmax(*dmax, hypot(v.x - (row == col ? 1.0 : 0.0), v.y));
      C[(long long)col * n + row] = v;
    }
  }
}

__global__ void __launch_bounds__(ND_THREADS) nd_persist_kernel(const NdParams p) {
  __shared__ double sh[ND_WARPS * 4];
  extern __shared__ double2 dsm[];
  cg::grid_group grid = cg::this_grid();
  const int n = p.n;
  const long long total = (long long)n * n;
  // first measurement straight from the input, which is copied to G0 in the
  // same pass (kept for the exact re-projection G = W^H G0 W)
  double2 *X = p.X, *W = p.W, *W2 = p.W2;
  build_phase(p.ain, p.lda, n, X, p.part, sh, p.G0);
  grid.sync();
  static_assert(kNumSMs <= ND_THREADS, "grid_max4 reads one CTA's partials per thread");
  double gm[4];
  grid_max4(p.part, gm, sh);
  double rmax = gm[0], emax = gm[1], dmax = gm[2];
  double last_defect = 0.0;
  bool done = false;
  int it = 0;
  for (;; ++it) {
    if (it > 0 && emax <= p.tol * fmax(1.0, dmax)) {
      done = last_defect <= 1e-8;  // W unitary to rounding, else zheevd
      break;
    }
    if (it == kNdMaxSteps || !(rmax <= p.bail)) break;  // not near-diagonal / not converging
    if (it == 0) {
      double2* tmp = W;  // W = X
      W = X;
      X = tmp;
    } else {
      gemm_phase<false>(W, X, W2, n, EPI_STORE, nullptr, nullptr, dsm);  // W X
      grid.sync();
      double2* tmp = W;
      W = W2;
      W2 = tmp;
    }
    // unitarity defect of W X ~ |S|^2 <~ (sqrt(n) r)^2, squared by each NS step
    const double sr = sqrt((double)n) * rmax;
    const int ns = sr <= 5e-5 ? 1 : (sr <= 7e-3 ? 2 : (sr <= 0.08 ? 3 : (sr <= 0.3 ? 4 : 5)));
    for (int k = 0; k < ns; ++k) {
      double dpart[4] = {0.0, 0.0, 0.0, 0.0};
      gemm_phase<true>(W, W, p.T, n, k == ns - 1 ? EPI_DEFECT : EPI_STORE, nullptr, &dpart[0], dsm);
      if (k == ns - 1) {
        double one[4] = {dpart[0], 0.0, 0.0, 0.0};
        block_max_publish(one, 1, 3, p.part, sh);
      }
      grid.sync();
      gemm_phase<false>(W, p.T, W2, n, EPI_NS, W, nullptr, dsm);  // 1.5 W - 0.5 W (W^H W)
      grid.sync();
      double2* tmp = W;
      W = W2;
      W2 = tmp;
    }
    gemm_phase<false>(p.G0, W, X, n, EPI_STORE, nullptr, nullptr, dsm);  // X = G0 W
    grid.sync();
    gemm_phase<true>(W, X, p.G, n, EPI_HERM, nullptr, nullptr, dsm);     // G = W^H G0 W
    grid.sync();
    build_phase(p.G, n, n, X, p.part, sh);
    grid.sync();
    grid_max4(p.part, gm, sh);
    rmax = gm[0];
    emax = gm[1];
    dmax = gm[2];
    last_defect = gm[3];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.status[0] = done ? 1.0 : 0.0;
    p.status[1] = (double)it;
    p.status[2] = rmax;
    p.status[3] = emax;
  }
  if (!done) return;  // grid-uniform
  // ascending eigenvalues (rank sort of the real diagonal, ties by index):
  // every CTA ranks the whole diagonal in shared memory (n <= 256: one entry
  // per thread), so the column gather needs no grid barrier after the sort
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  double* diag = reinterpret_cast<double*>(dsm);
  int* perm_s = reinterpret_cast<int*>(diag + kNdPersistMaxN);
  for (int i = threadIdx.x; i < n; i += blockDim.x) diag[i] = __ldcg(&p.G[(long long)i * n + i].x);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double di = diag[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = diag[j];
      rank += (dj < di) || (dj == di && j < i);
    }
    perm_s[rank] = i;
    if (blockIdx.x == 0) p.w[rank] = di;
  }
  __syncthreads();
  for (long long idx = gt; idx < total; idx += nt) {
    const int r = (int)(idx / n), i = (int)(idx % n);
    p.aout[(long long)r * p.lda + i] = __ldcg(&W[(long long)perm_s[r] * n + i]);
  }
}

}  // namespace

size_t nd_persist_ws_bytes(int n) {
  return 6 * (size_t)n * n * sizeof(double2) + (size_t)kNumSMs * 4 * sizeof(double) +
         (size_t)n * sizeof(int) + 4 * sizeof(double) + 1024;
}

// status_dev[0] = 1 when solved (A overwritten with the sorted eigenvectors,
// w with the eigenvalues), 0 when the caller must use zheevd (A untouched).
cudaError_t nd_persist_launch(const double2* a, long long lda, int n, double* w, double tol,
                              double bail, void* ws, double* status_dev, cudaStream_t s) {
  if (n < 2 || n > kNdPersistMaxN) return cudaErrorInvalidValue;
  NdParams p{};
  p.ain = a;
  p.lda = lda;
  p.aout = const_cast<double2*>(a);
  p.w = w;
  p.n = n;
  double2* base = static_cast<double2*>(ws);
  const size_t m = (size_t)n * n;
  p.G0 = base;
  p.G = base + m;
  p.X = base + 2 * m;
  p.T = base + 3 * m;
  p.W = base + 4 * m;
  p.W2 = base + 5 * m;
  p.part = reinterpret_cast<double*>(base + 6 * m);
  p.perm = reinterpret_cast<int*>(p.part + kNumSMs * 4);
  p.status = status_dev;
  p.tol = tol;
  p.bail = bail;
  // one CTA per 16x16 output tile of the products, at most one per SM
  const int t16 = (n + 15) / 16;
  int grid = t16 * t16;
  if (grid > kNumSMs) grid = kNumSMs;
  if (grid < 8) grid = 8;
  const size_t smem = nd_smem_doubles2(kNdPersistMaxN) * sizeof(double2);
  static const cudaError_t attr = cudaFuncSetAttribute(
      reinterpret_cast<const void*>(nd_persist_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)smem);
  if (attr != cudaSuccess) return attr;
  void* args[] = {&p};
  note_launch();
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(nd_persist_kernel), dim3(grid),
                                     dim3(ND_THREADS), args, nd_smem_doubles2(n) * sizeof(double2), s);
}

}  // namespace chfsi
