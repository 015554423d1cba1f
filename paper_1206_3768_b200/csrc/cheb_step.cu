// K1 — fused Chebyshev recurrence step on FP64 tensor cores (sm_100a).
//
//   Ynext = alpha * (H * Ycur - c * Ycur) - beta * Yprev
//
// restating one iteration of `chebyshev_filter` (reference
// spectral_chain/chfsi.py:202-207) as ONE kernel: the complex n x n x w
// product runs on DMMA.8x8x4 (mma.sync f64 — tcgen05 has no f64 kind), the
// shift, scale and three-term recurrence are applied in the epilogue while
// the accumulator tile is still in registers, and Ynext may alias Yprev so
// the whole filter ping-pongs between two n x w buffers.
//
// Layouts: H is read row-major (H[m*ldh + k], k contiguous); CONJ reads the
// conjugate, so a column-major Hermitian H (cuBLAS/cuSOLVER output) is used
// as-is. Y blocks are column-major (Y[col*ld + row]). complex128 interleaved.
//
// Tiling: CTA tile BM x BN (complex), K in slabs of BK=16 staged through a
// STAGES-deep cp.async ring in shared memory (pitch padded so the 16-byte
// fragment loads are bank-conflict free). Thin shapes (small w, small n) are
// split along K across a thread-block cluster; the partial tiles are summed
// in FIXED order through distributed shared memory, so the result is
// bitwise run-to-run reproducible (reference test_chfsi.py:234-241).
#include <cooperative_groups.h>

#include "chfsi_internal.h"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace chfsi {

constexpr int BK = 16;              // complex elements per K slab
constexpr int ROWB = BK * 16 + 64;  // smem row pitch (bytes); == 64 mod 128

struct ChebStepParams {
  const double2* h;
  long long ldh;
  const double2* ycur;
  long long ldc;
  const double2* yprev;
  long long ldp;
  double2* ynext;
  long long ldn;
  int n;        // rows of H and Y, also the contraction length
  int w;        // columns of Y
  int tiles_n;  // ceil(w / BN)
  int k_split;  // contraction extent of one split (multiple of BK)
  double alpha, c, beta;
  int read_cur;   // epilogue needs Ycur (c != 0)
  int read_prev;  // epilogue needs Yprev (beta != 0)
};

__device__ __forceinline__ void epilogue_store(const ChebStepParams& p, int row, int col, double ar,
                                               double ai) {
  double tr = ar, ti = ai;
  if (p.read_cur) {
    const double2 y = p.ycur[(long long)col * p.ldc + row];
    tr = dsub(tr, dmul(p.c, y.x));
    ti = dsub(ti, dmul(p.c, y.y));
  }
  tr = dmul(p.alpha, tr);
  ti = dmul(p.alpha, ti);
  double2* dst = p.ynext + (long long)col * p.ldn + row;
  if (p.read_prev) {
    const double2 yp = p.yprev[(long long)col * p.ldp + row];
    tr = dsub(tr, dmul(p.beta, yp.x));
    ti = dsub(ti, dmul(p.beta, yp.y));
  }
  *dst = make_double2(tr, ti);
}

template <int BM, int BN, int WM, int WN, int STAGES, bool CONJ, int SPLIT>
__global__ void __launch_bounds__(WM* WN * 32, 1) cheb_step_kernel(const ChebStepParams p) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int TM = BM / WM, TN = BN / WN;
  constexpr int MI = TM / 8, NI = TN / 8;
  constexpr int STAGE_BYTES = (BM + BN) * ROWB;
  static_assert(MI >= 1 && NI >= 1, "warp tile too small");
  static_assert(SPLIT == 1 || BM % SPLIT == 0, "split must divide BM");
  extern __shared__ __align__(128) unsigned char smem[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / WN, wn = warp % WN;
  const int tile = blockIdx.x / SPLIT;
  const int split = blockIdx.x % SPLIT;
  const int tm = tile / p.tiles_n, tn = tile % p.tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const int kbeg = split * p.k_split;
  const int kend = min(p.n, kbeg + p.k_split);
  const int nslab = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  double cr[MI][NI][2], ci[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

  auto load_slab = [&](int slab, int stage) {
    unsigned char* sa = smem + stage * STAGE_BYTES;
    unsigned char* sb = sa + BM * ROWB;
    const int k0 = kbeg + slab * BK;
#pragma unroll
    for (int it = 0; it < (BM * BK + THREADS - 1) / THREADS; ++it) {
      const int id = tid + it * THREADS;
      if (id < BM * BK) {
        const int r = id / BK, kk = id % BK;
        const int gm = m0 + r, gk = k0 + kk;
        const bool ok = gm < p.n && gk < kend;
        cp_async16(sa + r * ROWB + kk * 16, ok ? p.h + (long long)gm * p.ldh + gk : p.h, ok);
      }
    }
#pragma unroll
    for (int it = 0; it < (BN * BK + THREADS - 1) / THREADS; ++it) {
      const int id = tid + it * THREADS;
      if (id < BN * BK) {
        const int r = id / BK, kk = id % BK;
        const int gn = n0 + r, gk = k0 + kk;
        const bool ok = gn < p.w && gk < kend;
        cp_async16(sb + r * ROWB + kk * 16, ok ? p.ycur + (long long)gn * p.ldc + gk : p.ycur, ok);
      }
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nslab) load_slab(s, s);
    cp_async_commit();
  }

  for (int slab = 0; slab < nslab; ++slab) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = slab + STAGES - 1;
    if (nxt < nslab) load_slab(nxt, nxt % STAGES);
    cp_async_commit();

    const unsigned char* sa = smem + (slab % STAGES) * STAGE_BYTES + (wm * TM + g) * ROWB + t * 16;
    const unsigned char* sb = smem + (slab % STAGES) * STAGE_BYTES + BM * ROWB + (wn * TN + g) * ROWB + t * 16;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double2 a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = lds128(sa + i * 8 * ROWB + k4 * 64);
#pragma unroll
      for (int j = 0; j < NI; ++j) b[j] = lds128(sb + j * 8 * ROWB + k4 * 64);
      // Re/Im of (a or conj(a)) * b: four real DMMAs per complex 8x8x4 block.
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          dmma884(cr[i][j], a[i].x, b[j].x);
          dmma884(ci[i][j], a[i].x, b[j].y);
        }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const double ai = a[i].y, nai = -a[i].y;
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          dmma884(cr[i][j], CONJ ? ai : nai, b[j].y);
          dmma884(ci[i][j], CONJ ? nai : ai, b[j].x);
        }
      }
    }
  }
  cp_async_wait<0>();

  if constexpr (SPLIT == 1) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = m0 + wm * TM + i * 8 + g;
          const int col = n0 + wn * TN + j * 8 + 2 * t + e;
          if (row < p.n && col < p.w) epilogue_store(p, row, col, cr[i][j][e], ci[i][j][e]);
        }
  } else {
    // Deterministic split-K: stage the partial tile column-major in this
    // CTA's smem, then CTA r of the cluster sums rows [r*BM/S, (r+1)*BM/S)
    // over ranks 0..S-1 in order and applies the epilogue.
    constexpr int RP = BM + 2;  // column pitch (complex) of the partial tile
    static_assert(BN * RP * 16 <= STAGES * STAGE_BYTES, "partial tile does not fit");
    cg::cluster_group cluster = cg::this_cluster();
    __syncthreads();
    double2* red = reinterpret_cast<double2*>(smem);
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wm * TM + i * 8 + g;
          const int cidx = wn * TN + j * 8 + 2 * t + e;
          red[cidx * RP + r] = make_double2(cr[i][j][e], ci[i][j][e]);
        }
    cluster.sync();
    const int rank = static_cast<int>(cluster.block_rank());
    constexpr int RPER = BM / SPLIT;
    for (int idx = tid; idx < RPER * BN; idx += THREADS) {
      const int rr = rank * RPER + idx % RPER, cc = idx / RPER;
      const int row = m0 + rr, col = n0 + cc;
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int q = 0; q < SPLIT; ++q) {
        const double2* rem = cluster.map_shared_rank(red, q);
        const double2 v = rem[cc * RP + rr];
        sr = dadd(sr, v.x);
        si = dadd(si, v.y);
      }
      if (row < p.n && col < p.w) epilogue_store(p, row, col, sr, si);
    }
    cluster.sync();
  }
}

// ------------------------------------------------------------------ host ---

namespace {

template <int BM, int BN, int WM, int WN, int STAGES, bool CONJ, int SPLIT>
cudaError_t launch_cfg(const ChebStepParams& p0, int tiles_m, cudaStream_t stream) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int SMEM = STAGES * (BM + BN) * ROWB;
  auto kern = cheb_step_kernel<BM, BN, WM, WN, STAGES, CONJ, SPLIT>;
  static bool attr_set = false;  // per template instance
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  ChebStepParams p = p0;
  p.tiles_n = (p.w + BN - 1) / BN;
  const int kper = (p.n + SPLIT - 1) / SPLIT;
  p.k_split = ((kper + BK - 1) / BK) * BK;
  const int ctas = tiles_m * p.tiles_n * SPLIT;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas, 1, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = SPLIT;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int BM, int BN, int WM, int WN, int STAGES, bool CONJ>
cudaError_t launch_split(const ChebStepParams& p, int split, cudaStream_t s) {
  const int tiles_m = (p.n + BM - 1) / BM;
  switch (split) {
    case 1: return launch_cfg<BM, BN, WM, WN, STAGES, CONJ, 1>(p, tiles_m, s);
    case 2: return launch_cfg<BM, BN, WM, WN, STAGES, CONJ, 2>(p, tiles_m, s);
    case 4: return launch_cfg<BM, BN, WM, WN, STAGES, CONJ, 4>(p, tiles_m, s);
    case 8: return launch_cfg<BM, BN, WM, WN, STAGES, CONJ, 8>(p, tiles_m, s);
    default: return cudaErrorInvalidValue;
  }
}

// Modelled cost (in MAC-slab units) of one launch: waves x per-CTA work,
// plus the fixed pipeline fill and the split reduction.
double model_cost(int n, int w, int bm, int bn, int split) {
  const long long tiles = (long long)((n + bm - 1) / bm) * ((w + bn - 1) / bn);
  const long long ctas = tiles * split;
  const long long waves = (ctas + kNumSMs - 1) / kNumSMs;
  const int kper = (((n + split - 1) / split + BK - 1) / BK) * BK;
  const double per_cta = (double)bm * bn * (kper + 3.0 * BK) + (split > 1 ? 4.0 * bm * bn * split : 0.0);
  return waves * per_cta;
}

}  // namespace

StepTiling choose_step_tiling(int n, int w) {
  StepTiling best{64, 64, 1};
  double best_cost = 1e300;
  const int bns[2] = {64, 32};
  const int splits[4] = {1, 2, 4, 8};
  for (int bn : bns)
    for (int s : splits) {
      if (s > 1 && (n + s - 1) / s < 2 * BK) continue;
      const double c = model_cost(n, w, 64, bn, s) * (bn == 32 ? 1.04 : 1.0);
      if (c < best_cost) {
        best_cost = c;
        best = StepTiling{64, bn, s};
      }
    }
  return best;
}

cudaError_t cheb_step_launch(const double2* h, long long ldh, bool conj_h, const double2* ycur,
                             long long ldc, const double2* yprev, long long ldp, double2* ynext,
                             long long ldn, int n, int w, double alpha, double c, double beta,
                             StepTiling tiling, cudaStream_t stream) {
  if (n <= 0 || w <= 0) return cudaSuccess;
  ChebStepParams p{};
  p.h = h;
  p.ldh = ldh;
  p.ycur = ycur;
  p.ldc = ldc;
  p.yprev = yprev ? yprev : ynext;
  p.ldp = yprev ? ldp : ldn;
  p.ynext = ynext;
  p.ldn = ldn;
  p.n = n;
  p.w = w;
  p.alpha = alpha;
  p.c = c;
  p.beta = beta;
  p.read_cur = c != 0.0;
  p.read_prev = (beta != 0.0) && yprev != nullptr;
  if (tiling.bm == 0) tiling = choose_step_tiling(n, w);
  if (tiling.bm != 64) return cudaErrorInvalidValue;
  if (tiling.bn == 64)
    return conj_h ? launch_split<64, 64, 2, 4, 4, true>(p, tiling.split, stream)
                  : launch_split<64, 64, 2, 4, 4, false>(p, tiling.split, stream);
  if (tiling.bn == 32)
    return conj_h ? launch_split<64, 32, 4, 2, 4, true>(p, tiling.split, stream)
                  : launch_split<64, 32, 4, 2, 4, false>(p, tiling.split, stream);
  return cudaErrorInvalidValue;
}

}  // namespace chfsi
