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
// Schedule: a persistent grid of exactly the resident CTAs (2 per SM) walks
// a linearised (tile, k-slab) iteration space — whole tiles first
// ("data-parallel" waves, consecutive CTAs on neighbouring column tiles of
// one H row panel so the panel is shared through L2), then the remaining
// tiles split evenly across all CTAs by k-slab ("stream-K"). A tile whose
// k-range is split is finished by the CTA holding its last slab: it waits
// for its peers' published partial tiles and sums them in FIXED peer order,
// so every launch is bitwise reproducible (reference test_chfsi.py:234-241)
// and no SM idles on a wave tail, whatever (n, w) the locking leaves.
//
// Pipeline: K slabs of BK=16 complex staged global->shared with a
// STAGES-deep cp.async ring; 16-byte chunks XOR-swizzled on row parity so
// the per-lane 16-byte fragment loads (8 rows x 4 k) are bank-conflict free.
#include <cstdint>

#include "chfsi_internal.h"
#include "common.cuh"

namespace chfsi {

namespace {

constexpr int BK = 16;             // complex elements per K slab
constexpr int ROWB = BK * 16;      // 256-byte smem rows (swizzled, no padding)
constexpr int kMaxThreads = 256;
constexpr int kMaxAcc = 32;        // doubles per thread in a partial tile (upper bound)

struct StepParams {
  const double2* h;
  long long ldh;
  const double2* ycur;
  long long ldc;
  const double2* yprev;
  long long ldp;
  double2* ynext;
  long long ldn;
  int n, w;
  int tiles_n;
  int kiters;          // K slabs per tile
  int dp_waves;        // whole tiles per CTA before the stream-K part
  int sk_first;        // first stream-K tile
  long long sk_iters;  // stream-K iterations (tiles * kiters)
  int sk_ctas;         // CTAs sharing the stream-K part (<= grid)
  double alpha, c, beta;
  int read_cur, read_prev;
  double* partials;    // [grid][ACC][THREADS]
  unsigned* flags;     // [grid]
  unsigned epoch;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void epilogue_store(const StepParams& p, int row, int col, double ar,
                                               double ai) {
  double tr = ar, ti = ai;
  if (p.read_cur) {
    const double2 y = p.ycur[(long long)col * p.ldc + row];
    tr = dsub(tr, dmul(p.c, y.x));
    ti = dsub(ti, dmul(p.c, y.y));
  }
  tr = dmul(p.alpha, tr);
  ti = dmul(p.alpha, ti);
  if (p.read_prev) {
    const double2 yp = p.yprev[(long long)col * p.ldp + row];
    tr = dsub(tr, dmul(p.beta, yp.x));
    ti = dsub(ti, dmul(p.beta, yp.y));
  }
  p.ynext[(long long)col * p.ldn + row] = make_double2(tr, ti);
}

// byte offset of 16-byte chunk `kk` of smem row `r` (row-parity XOR swizzle)
__device__ __forceinline__ int swz(int r, int kk) { return r * ROWB + ((kk ^ ((r & 1) << 2)) << 4); }

template <int BM, int BN, int WM, int WN, int STAGES, int MINB, bool CONJ>
__global__ void __launch_bounds__(WM* WN * 32, MINB) cheb_step_kernel(const StepParams p) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int TM = BM / WM, TN = BN / WN;
  constexpr int MI = TM / 8, NI = TN / 8;
  constexpr int ACC = MI * NI * 4;
  constexpr int STAGE_BYTES = (BM + BN) * ROWB;
  static_assert(THREADS <= kMaxThreads && ACC <= kMaxAcc, "workspace bound");
  static_assert((BM * BK) % THREADS == 0, "A-tile copy split");
  static_assert(MI >= 1 && NI >= 1, "warp tile too small");
  extern __shared__ __align__(128) unsigned char smem[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / WN, wn = warp % WN;
  const int G = gridDim.x, cta = blockIdx.x;
  const int kiters = p.kiters;

  // ---- this CTA's slice of the linearised iteration space (64-bit once)
  const int dp_iters = p.dp_waves * kiters;
  int sb = 0, se = 0;
  if (cta < p.sk_ctas) {
    sb = (int)((long long)cta * p.sk_iters / p.sk_ctas);
    se = (int)((long long)(cta + 1) * p.sk_iters / p.sk_ctas);
  }
  const int total = dp_iters + (se - sb);
  if (total == 0) return;
  // If the range ends inside a tile, that head-of-tile segment is a partial
  // the tile's owner (a later CTA) will consume: compute and publish it
  // FIRST, so owners never wait on a chain of peers. Local order:
  //   [publish segment] [data-parallel tiles] [rest of the stream-K range]
  int pub = 0;
  if (se > sb && (se % kiters) != 0) {
    const int head = ((se - 1) / kiters) * kiters;
    pub = se - (head > sb ? head : sb);
  }
  const int sk_tile0 = p.sk_first + sb / kiters, sk_kk0 = sb % kiters;

  // Cursor over that order; advanced incrementally (no per-slab division).
  struct Cursor {
    int j, tile, kk, m0, n0;
  };
  auto set_tile = [&](Cursor& c, int tile, int kk) {
    c.tile = tile;
    c.kk = kk;
    c.m0 = (tile / p.tiles_n) * BM;
    c.n0 = (tile % p.tiles_n) * BN;
  };
  auto start = [&](Cursor& c) {
    c.j = 0;
    if (pub > 0) {
      const int s0 = se - pub;
      set_tile(c, p.sk_first + s0 / kiters, s0 % kiters);
    } else if (dp_iters > 0) {
      set_tile(c, cta, 0);
    } else {
      set_tile(c, sk_tile0, sk_kk0);
    }
  };
  auto advance = [&](Cursor& c) {
    ++c.j;
    ++c.kk;
    if (pub > 0 && c.j == pub) {
      if (dp_iters > 0) set_tile(c, cta, 0);
      else set_tile(c, sk_tile0, sk_kk0);
    } else if (dp_iters > 0 && c.j == pub + dp_iters) {
      set_tile(c, sk_tile0, sk_kk0);
    } else if (c.kk == kiters) {
      set_tile(c, c.tile + ((c.j < pub + dp_iters) ? G : 1), 0);
    }
  };

  // per-thread global->smem copy coordinates (fixed for the whole kernel)
  const int lrow = tid / BK, lcol = tid % BK;  // row lrow + it*(THREADS/BK), 16-byte chunk lcol
  auto load_iter = [&](const Cursor& c, int stage) {
    const int k0 = c.kk * BK + lcol;
    unsigned char* sa = smem + stage * STAGE_BYTES;
    unsigned char* sbuf = sa + BM * ROWB;
    const bool kok = k0 < p.n;
#pragma unroll
    for (int it = 0; it < (BM * BK) / THREADS; ++it) {
      const int r = lrow + it * (THREADS / BK);
      const int gm = c.m0 + r;
      const bool ok = kok && gm < p.n;
      cp_async16(sa + swz(r, lcol), ok ? p.h + (long long)gm * p.ldh + k0 : p.h, ok);
    }
#pragma unroll
    for (int it = 0; it < (BN * BK + THREADS - 1) / THREADS; ++it) {
      const int r = lrow + it * (THREADS / BK);
      if ((BN * BK) % THREADS == 0 || r < BN) {
        const int gn = c.n0 + r;
        const bool ok = kok && gn < p.w;
        cp_async16(sbuf + swz(r, lcol), ok ? p.ycur + (long long)gn * p.ldc + k0 : p.ycur, ok);
      }
    }
  };

  double acc[MI][NI][4];  // [.][.][0..1] real, [2..3] imag of C[g][2t+e]
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  auto epilogue = [&](const Cursor& c) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = c.m0 + wm * TM + i * 8 + g;
          const int col = c.n0 + wn * TN + j * 8 + 2 * t + e;
          if (row < p.n && col < p.w) epilogue_store(p, row, col, acc[i][j][e], acc[i][j][2 + e]);
        }
  };

  Cursor lc;
  start(lc);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (lc.j < total) {
      load_iter(lc, s);
      advance(lc);
    }
    cp_async_commit();
  }

  // fragment addresses: rows arow+8i / brow+8j, chunk (k4*4 + t) ^ swizzle
  const int arow = wm * TM + g, brow = wn * TN + g;
  Cursor cc;
  start(cc);
  for (int j = 0; j < total; ++j) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (lc.j < total) {
      load_iter(lc, lc.j % STAGES);
      advance(lc);
    }
    cp_async_commit();

    const unsigned char* sa = smem + (j % STAGES) * STAGE_BYTES;
    const unsigned char* sbm = sa + BM * ROWB;
    double2 a[2][MI], b[2][NI];
#pragma unroll
    for (int i = 0; i < MI; ++i) a[0][i] = lds128(sa + swz(arow + i * 8, t));
#pragma unroll
    for (int jj = 0; jj < NI; ++jj) b[0][jj] = lds128(sbm + swz(brow + jj * 8, t));
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int cur = k4 & 1, nxt = cur ^ 1;
      if (k4 + 1 < BK / 4) {  // prefetch the next k4 fragments (software pipeline)
#pragma unroll
        for (int i = 0; i < MI; ++i) a[nxt][i] = lds128(sa + swz(arow + i * 8, (k4 + 1) * 4 + t));
#pragma unroll
        for (int jj = 0; jj < NI; ++jj)
          b[nxt][jj] = lds128(sbm + swz(brow + jj * 8, (k4 + 1) * 4 + t));
      }
      // Re/Im of (a or conj(a)) * b: four real DMMAs per complex 8x8x4 block
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int jj = 0; jj < NI; ++jj) {
          double(&cr)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][0]);
          double(&ci)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][2]);
          dmma884(cr, a[cur][i].x, b[cur][jj].x);
          dmma884(ci, a[cur][i].x, b[cur][jj].y);
        }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const double ai = a[cur][i].y, nai = -a[cur][i].y;
#pragma unroll
        for (int jj = 0; jj < NI; ++jj) {
          double(&cr)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][0]);
          double(&ci)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][2]);
          dmma884(cr, CONJ ? ai : nai, b[cur][jj].y);
          dmma884(ci, CONJ ? nai : ai, b[cur][jj].x);
        }
      }
    }

    // ---- end of a tile segment?
    const bool tile_end = cc.kk == kiters - 1;
    const bool pub_end = pub > 0 && j == pub - 1;
    if (tile_end || pub_end) {
      if (pub_end) {
        // non-owner: publish the partial head of this CTA's last tile
        double* dst = p.partials + (size_t)cta * ACC * THREADS + tid;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < NI; ++jj)
#pragma unroll
            for (int e = 0; e < 4; ++e) __stcg(dst + ((i * NI + jj) * 4 + e) * THREADS, acc[i][jj][e]);
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release(p.flags + cta, p.epoch);
      } else if (j < pub + dp_iters) {
        epilogue(cc);
      } else {
        const int tile_s0 = (cc.tile - p.sk_first) * kiters;  // first SK iteration of the tile
        if (tile_s0 >= sb) {
          epilogue(cc);
        } else {
          // owner: the peers are the CTAs whose ranges hold [tile_s0, sb)
          const int first =
              (int)(((long long)(tile_s0 + 1) * p.sk_ctas + p.sk_iters - 1) / p.sk_iters) - 1;
          if (tid == 0) {
            for (int q = first; q < cta; ++q)
              while (ld_acquire(p.flags + q) != p.epoch) __nanosleep(64);
          }
          __syncthreads();
          // fixed fold order: own partial, then peers first..cta-1
          for (int q = first; q < cta; ++q) {
            const double* src = p.partials + (size_t)q * ACC * THREADS + tid;
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
              for (int jj = 0; jj < NI; ++jj)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  acc[i][jj][e] = dadd(acc[i][jj][e], __ldcg(src + ((i * NI + jj) * 4 + e) * THREADS));
          }
          epilogue(cc);
        }
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int jj = 0; jj < NI; ++jj)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[i][jj][e] = 0.0;
    }
    advance(cc);
  }
  cp_async_wait<0>();
}

// --------------------------------------------------------------- host ---

struct Variant {
  const void* fn;
  int bm, bn, threads, smem;
  int resident;  // CTAs per SM actually achievable
};

template <int BM, int BN, int WM, int WN, int STAGES, int MINB, bool CONJ>
Variant make_variant() {
  Variant v{};
  auto fn = cheb_step_kernel<BM, BN, WM, WN, STAGES, MINB, CONJ>;
  v.fn = reinterpret_cast<const void*>(fn);
  v.bm = BM;
  v.bn = BN;
  v.threads = WM * WN * 32;
  v.smem = STAGES * (BM + BN) * ROWB;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v.smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, v.threads, v.smem);
  v.resident = occ > 0 ? occ : 1;
  return v;
}

// (bm, bn) -> kernel configuration. Function-local statics: built once, on
// first use (the caller has set the device).
const Variant* variant(int bm, int bn, bool conj) {
#define CHFSI_V(BM_, BN_, WM_, WN_, ST_, MB_)                                         \
  if (bm == BM_ && bn == BN_) {                                                       \
    static const Variant a = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, false>();     \
    static const Variant b = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, true>();      \
    return conj ? &b : &a;                                                            \
  }
  CHFSI_V(64, 16, 8, 1, 4, 2)
  CHFSI_V(64, 32, 4, 2, 4, 2)
  CHFSI_V(64, 64, 2, 4, 3, 2)
  CHFSI_V(32, 32, 2, 2, 4, 3)
  CHFSI_V(32, 64, 2, 2, 3, 3)
  CHFSI_V(128, 32, 4, 2, 3, 1)
#undef CHFSI_V
  return nullptr;
}

}  // namespace

StepTiling choose_step_tiling(int n, int w) {
  // least padded work, mild preference for wider tiles (operand reuse)
  const int bns[3] = {64, 32, 16};
  const double pen[3] = {1.0, 1.03, 1.10};
  StepTiling best{64, 64, 0};
  double best_cost = 1e300;
  for (int i = 0; i < 3; ++i) {
    const double padded = (double)((w + bns[i] - 1) / bns[i]) * bns[i];
    const double cost = padded * pen[i];
    if (cost < best_cost) {
      best_cost = cost;
      best = StepTiling{64, bns[i], 0};
    }
  }
  (void)n;
  return best;
}

size_t step_workspace_doubles(int max_grid) { return (size_t)max_grid * kMaxAcc * kMaxThreads; }

int step_grid_size(int bn, bool conj) {
  const Variant* v = variant(64, bn, conj);
  return v ? v->resident * kNumSMs : 0;
}

cudaError_t cheb_step_launch(const double2* h, long long ldh, bool conj_h, const double2* ycur,
                             long long ldc, const double2* yprev, long long ldp, double2* ynext,
                             long long ldn, int n, int w, double alpha, double c, double beta,
                             StepTiling tiling, const StepWorkspace& ws, cudaStream_t stream) {
  if (n <= 0 || w <= 0) return cudaSuccess;
  if (tiling.bm == 0) tiling = choose_step_tiling(n, w);
  const Variant* vp = variant(tiling.bm, tiling.bn, conj_h);
  if (vp == nullptr) return cudaErrorInvalidValue;
  const Variant& v = *vp;
  const int BM = v.bm;
  int grid = v.resident * kNumSMs;
  if (tiling.split > 0 && tiling.split < grid) grid = tiling.split;  // test/tuning override
  if (grid > ws.max_grid) return cudaErrorInvalidValue;

  StepParams p{};
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
  p.tiles_n = (w + tiling.bn - 1) / tiling.bn;
  const int tiles_m = (n + BM - 1) / BM;
  const long long tiles = (long long)tiles_m * p.tiles_n;
  p.kiters = (n + BK - 1) / BK;
  p.dp_waves = tiles >= 2LL * grid ? (int)(tiles / grid) - 1 : 0;
  p.sk_first = p.dp_waves * grid;
  p.sk_iters = (tiles - p.sk_first) * p.kiters;
  p.sk_ctas = (int)(p.sk_iters < grid ? p.sk_iters : grid);
  p.alpha = alpha;
  p.c = c;
  p.beta = beta;
  p.read_cur = c != 0.0;
  p.read_prev = (beta != 0.0) && yprev != nullptr;
  p.partials = ws.partials;
  p.flags = ws.flags;
  p.epoch = ++*ws.epoch;
  void* args[] = {&p};
  note_launch();
  return cudaLaunchKernel(v.fn, dim3(grid), dim3(v.threads), args, v.smem, stream);
}

}  // namespace chfsi
