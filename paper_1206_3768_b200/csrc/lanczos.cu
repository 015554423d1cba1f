// K2 — the whole k-step Lanczos bound (reference chfsi.py:125-162) as ONE
// cooperative persistent kernel.
//
// Per step: u = H q (HBM-bound GEMV, each block its own row range),
// alpha = Re(q^H u), r = u - alpha q - beta q_prev, full reorthogonalisation
// r -= V (V^H r), beta = ||r||, q_next = r / beta, with the breakdown test
// beta < 1e-14 of chfsi.py:152. Four grid-wide barriers per step replace the
// nine kernel launches of the multi-kernel version (launch latency dominated
// it below n ~ 5000). Every reduction uses a fixed partition and a fixed
// combining order (block partials summed in block order), so alphas/betas are
// bitwise reproducible run to run.
#include <cooperative_groups.h>

#include "chfsi_internal.h"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace chfsi {

namespace {

constexpr int LZ_THREADS = 512;
constexpr int LZ_WARPS = LZ_THREADS / 32;

struct LanczosParams {
  const double2* h;
  long long ldh;
  int n, k;
  const double2* q0;  // raw start vector (normalised here)
  double2* V;         // n x k basis, column-major, ld n
  double2* u;         // n
  double2* r;         // n
  double* part;       // [2][grid] scalar partials: alpha (and ||q0||^2) in [0, G), beta in [G, 2G)
  double2* cpart;     // [grid][k] reorthogonalisation partials
  double2* coef;      // [k]
  double* alphas;     // [k]
  double* betas;      // [k]
  LanczosState* st;
  int cache_h;        // H fits in L2: cached loads (re-read every step) instead of streaming
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// fixed-tree block sum, result broadcast to every thread
__device__ double block_sum_all(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < LZ_WARPS ? sh[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) sh[LZ_WARPS] = r;
  }
  __syncthreads();
  r = sh[LZ_WARPS];
  __syncthreads();
  return r;
}

// sum of the G block partials in block order (every block gets the same bits)
__device__ double grid_total(const double* part, int G, double* sh) {
  double v = 0.0;
  for (int b = threadIdx.x; b < G; b += LZ_THREADS) v += __ldcg(part + b);
  return block_sum_all(v, sh);
}

template <bool CONJ>
__global__ void __launch_bounds__(LZ_THREADS) lanczos_coop_kernel(const LanczosParams p) {
  __shared__ double sh[LZ_WARPS + 1];
  __shared__ double2 red[LZ_THREADS];  // (row, j-group) partials of r -= V coef
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int r0 = (int)((long long)n * b / G), r1 = (int)((long long)n * (b + 1) / G);

  // ---- q = q0 / ||q0||  (chfsi.py:137-138)
  double s = 0.0;
  for (int i = r0 + tid; i < r1; i += LZ_THREADS) {
    const double2 x = p.q0[i];
    s = fma(x.x, x.x, fma(x.y, x.y, s));
  }
  s = block_sum_all(s, sh);
  if (tid == 0) p.part[b] = s;
  grid.sync();
  const double nq = sqrt(grid_total(p.part, G, sh));
  for (int i = r0 + tid; i < r1; i += LZ_THREADS) {
    const double2 x = p.q0[i];
    p.V[i] = make_double2(__ddiv_rn(x.x, nq), __ddiv_rn(x.y, nq));
  }
  grid.sync();

  double beta_prev = 0.0;
  for (int it = 0; it < p.k; ++it) {
    const double2* q = p.V + (long long)it * n;
    // The GEMV input: q itself at it = 0; afterwards the complete r of the
    // previous step scaled by 1/beta (q = r / beta is written by each block
    // for its own rows only, so reading r saves the grid barrier that would
    // otherwise publish q before the GEMV).
    const double2* gq = it ? p.r : q;
    const double gscale = it ? 1.0 / beta_prev : 1.0;
    // ---- u = H q on this block's rows (warp per row), alpha partial
    double ap = 0.0;
    for (int row = r0 + warp; row < r1; row += LZ_WARPS) {
      const double2* hr = p.h + (long long)row * p.ldh;
      double sr = 0.0, si = 0.0;
      int c = lane;
      const double sg = CONJ ? -1.0 : 1.0;
      // 8 independent 16-byte loads of H per lane in flight (HBM-bound GEMV:
      // the bytes in flight per SM set the bandwidth)
      for (; c + 224 < n; c += 256) {
        double2 a[8], bq[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)  // streamed once per step, or kept in L2 when it fits
          a[u] = p.cache_h ? __ldcg(hr + c + 32 * u) : __ldcs(hr + c + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) bq[u] = gq[c + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          sr = fma(a[u].x, bq[u].x, fma(-sg * a[u].y, bq[u].y, sr));
          si = fma(a[u].x, bq[u].y, fma(sg * a[u].y, bq[u].x, si));
        }
      }
      for (; c < n; c += 32) {
        const double2 a = hr[c], bb = gq[c];
        sr = fma(a.x, bb.x, fma(-sg * a.y, bb.y, sr));
        si = fma(a.x, bb.y, fma(sg * a.y, bb.x, si));
      }
      sr = warp_sum(sr) * gscale;
      si = warp_sum(si) * gscale;
      if (lane == 0) {
        p.u[row] = make_double2(sr, si);
        const double2 qv = q[row];
        ap = fma(qv.x, sr, fma(qv.y, si, ap));  // Re(conj(q) u)
      }
    }
    ap = block_sum_all(ap, sh);
    if (tid == 0) p.part[b] = ap;
    grid.sync();  // (1) alpha partials

    const double alpha = grid_total(p.part, G, sh);
    if (b == 0 && tid == 0) p.alphas[it] = alpha;
    // ---- r = (u - alpha q) - beta_prev q_prev on own rows
    const double2* qp = it ? p.V + (long long)(it - 1) * n : nullptr;
    for (int i = r0 + tid; i < r1; i += LZ_THREADS) {
      const double2 uu = p.u[i], qq = q[i];
      double rr = dsub(uu.x, dmul(alpha, qq.x)), ri = dsub(uu.y, dmul(alpha, qq.y));
      if (qp) {
        const double2 pp = qp[i];
        rr = dsub(rr, dmul(beta_prev, pp.x));
        ri = dsub(ri, dmul(beta_prev, pp.y));
      }
      p.r[i] = make_double2(rr, ri);
    }
    __syncthreads();
    // ---- reorthogonalisation partials: cpart[b][j] = V[own rows, j]^H r,
    // one thread per column j (each reads its column's contiguous row range)
    for (int j = tid; j <= it; j += LZ_THREADS) {
      const double2* vj = p.V + (long long)j * n;
      double cr = 0.0, ci = 0.0;
      int i = r0;
      for (; i + 3 < r1; i += 4) {  // four rows' loads in flight (same summation order)
        double2 a[4], rv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = vj[i + u];
          rv[u] = p.r[i + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cr = fma(a[u].x, rv[u].x, fma(a[u].y, rv[u].y, cr));
          ci = fma(a[u].x, rv[u].y, fma(-a[u].y, rv[u].x, ci));
        }
      }
      for (; i < r1; ++i) {
        const double2 a = vj[i], rv = p.r[i];
        cr = fma(a.x, rv.x, fma(a.y, rv.y, cr));
        ci = fma(a.x, rv.y, fma(-a.y, rv.x, ci));
      }
      p.cpart[(long long)b * p.k + j] = make_double2(cr, ci);
    }
    grid.sync();  // (2) partials complete

    // ---- coef[j] = sum_b cpart[b][j] (block order), j spread over warps
    for (int j = b * LZ_WARPS + warp; j <= it; j += G * LZ_WARPS) {
      double cr = 0.0, ci = 0.0;
      int bb = lane;
      for (; bb + 96 < G; bb += 128) {  // four blocks' partials in flight per lane (same order)
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcg(p.cpart + (long long)(bb + 32 * u) * p.k + j);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cr += v[u].x;
          ci += v[u].y;
        }
      }
      for (; bb < G; bb += 32) {
        const double2 v = __ldcg(p.cpart + (long long)bb * p.k + j);
        cr += v.x;
        ci += v.y;
      }
      cr = warp_sum(cr);
      ci = warp_sum(ci);
      if (lane == 0) p.coef[j] = make_double2(cr, ci);
    }
    grid.sync();  // (3) coefficients complete

    // ---- r -= V coef, beta partial. Threads split as (row, j-group): RP
    // rows x JG groups, each group summing a strided subset of the columns;
    // the JG partial sums are combined in group order (deterministic).
    double bp = 0.0;
    const int rows = r1 - r0;
    if (rows <= LZ_THREADS) {
      int rp = 1;
      while (rp < rows) rp <<= 1;
      const int jg = LZ_THREADS / rp;
      const int ri = tid % rp, gi = tid / rp;
      double sr = 0.0, si = 0.0;
      if (ri < rows) {
        const int i = r0 + ri;
        for (int j = gi; j <= it; j += jg) {
          const double2 a = p.V[(long long)j * n + i], c = __ldcg(p.coef + j);
          sr = fma(a.x, c.x, fma(-a.y, c.y, sr));
          si = fma(a.x, c.y, fma(a.y, c.x, si));
        }
      }
      red[tid] = make_double2(sr, si);
      __syncthreads();
      if (tid < rows) {
        double tr = 0.0, ti = 0.0;
        for (int gg = 0; gg < jg; ++gg) {
          const double2 v = red[gg * rp + tid];
          tr += v.x;
          ti += v.y;
        }
        const double2 rv = p.r[r0 + tid];
        const double2 nr = make_double2(rv.x - tr, rv.y - ti);
        p.r[r0 + tid] = nr;
        bp = fma(nr.x, nr.x, fma(nr.y, nr.y, bp));
      }
      __syncthreads();
    } else {  // very tall blocks: one thread per row, fixed j order
      for (int i = r0 + tid; i < r1; i += LZ_THREADS) {
        double sr = 0.0, si = 0.0;
        for (int j = 0; j <= it; ++j) {
          const double2 a = p.V[(long long)j * n + i], c = __ldcg(p.coef + j);
          sr = fma(a.x, c.x, fma(-a.y, c.y, sr));
          si = fma(a.x, c.y, fma(a.y, c.x, si));
        }
        const double2 rv = p.r[i];
        const double2 nr = make_double2(rv.x - sr, rv.y - si);
        p.r[i] = nr;
        bp = fma(nr.x, nr.x, fma(nr.y, nr.y, bp));
      }
    }
    bp = block_sum_all(bp, sh);
    // beta partials in their own half: a block leaving barrier (4) early
    // writes its next alpha partial into [0, G) while a lagging block may
    // still be summing these (single-buffered, that mixed alpha and beta
    // partials and gave blocks different betas)
    if (tid == 0) p.part[G + b] = bp;
    grid.sync();  // (4) beta partials

    const double beta = sqrt(grid_total(p.part + G, G, sh));
    const bool stop = (beta < 1e-14) || (it == p.k - 1);  // chfsi.py:152
    if (b == 0 && tid == 0) {
      p.st->steps = it + 1;
      p.st->beta_last = beta;
      if (stop) p.st->done = 1;
      else p.betas[it] = beta;
    }
    if (stop) break;
    double2* qn = p.V + (long long)(it + 1) * n;
    for (int i = r0 + tid; i < r1; i += LZ_THREADS) {
      const double2 x = p.r[i];
      qn[i] = make_double2(__ddiv_rn(x.x, beta), __ddiv_rn(x.y, beta));
    }
    beta_prev = beta;
    // q_next's rows are read by other threads of this block (lane 0 of the
    // row's warp, alpha partial of the next GEMV)
    __syncthreads();
    // no grid barrier: the next GEMV reads r (complete since barrier (4)), and r
    // is rewritten only after the next barrier (1)
  }
}

}  // namespace

size_t lanczos_coop_workspace_bytes(int n, int k) {
  const int G = lanczos_coop_grid(n);
  return 2 * (size_t)n * sizeof(double2) + 2 * (size_t)G * sizeof(double) +
         (size_t)G * k * sizeof(double2) + (size_t)k * sizeof(double2) + 256;
}

int lanczos_coop_grid(int n) {
  static int full = [] {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lanczos_coop_kernel<false>, LZ_THREADS, 0);
    int occ2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, lanczos_coop_kernel<true>, LZ_THREADS, 0);
    if (occ2 < occ) occ = occ2;
    if (occ > 2) occ = 2;  // enough bytes in flight for the GEMV; fewer partials
    return (occ > 0 ? occ : 1) * kNumSMs;
  }();
  // small n: the grid barriers dominate and one block per SM is cheaper
  // (measured at n = 2048: 37 vs 41 us per step; n = 5000 prefers 2 per SM)
  return n <= 3000 ? kNumSMs : full;
}

cudaError_t lanczos_coop_launch(const double2* h, long long ldh, bool conj_h, int n, int k,
                                const double2* q0, double2* V, void* ws, double* alphas,
                                double* betas, LanczosState* st, cudaStream_t s) {
  const int G = lanczos_coop_grid(n);
  LanczosParams p{};
  p.h = h;
  p.ldh = ldh;
  p.n = n;
  p.k = k;
  p.q0 = q0;
  p.V = V;
  char* base = static_cast<char*>(ws);
  p.u = reinterpret_cast<double2*>(base);
  p.r = p.u + n;
  p.cpart = p.r + n;
  p.coef = p.cpart + (size_t)G * k;
  p.part = reinterpret_cast<double*>(p.coef + k);
  p.alphas = alphas;
  p.betas = betas;
  p.st = st;
  // H re-read by every step: up to 100 MB (n <= 2560; L2 is 126 MB in two
  // halves) cache it in L2 instead of streaming it from HBM each step
  static const long long cache_limit = [] {
    const char* e = getenv("CHFSI_LZ_CACHE_BYTES");
    return e ? atoll(e) : 100LL << 20;  // n = 2048: cold k = 204 chain 8.2 -> 6.6 ms
  }();
  p.cache_h = 16LL * n * n <= cache_limit;
  void* args[] = {&p};
  note_launch();
  if (conj_h)
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lanczos_coop_kernel<true>),
                                       dim3(G), dim3(LZ_THREADS), args, 0, s);
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lanczos_coop_kernel<false>),
                                     dim3(G), dim3(LZ_THREADS), args, 0, s);
}

}  // namespace chfsi
