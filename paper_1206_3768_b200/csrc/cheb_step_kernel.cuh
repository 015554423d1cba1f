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
// Operand staging: TMA (cp.async.bulk.tensor, one elected thread) streams
// BK=16-complex k-slabs of the H row panel and of the Y column panel into a
// STAGES-deep shared-memory ring, completion tracked by mbarriers (full: TMA
// bytes landed; empty: all warps done reading). Each 256-byte k-row is split
// in two 128-byte TMA boxes with the hardware 128B swizzle; fragment rows are
// permuted inside each 8-row group (sigma) so the per-lane 16-byte fragment
// loads are bank-conflict free under that swizzle. Out-of-range rows,
// columns and k are zero-filled by the TMA unit (no predication in the loop).
//
// Schedule: a persistent grid of exactly the resident CTAs walks a
// linearised (tile, k-slab) iteration space — whole tiles in data-parallel
// waves (consecutive CTAs on neighbouring column tiles of one H row panel,
// so the panel is read from HBM once and reused through L2), the remaining
// tiles split evenly by k-slab ("stream-K"). A split tile is finished by the
// CTA holding its last slab, which waits for the peers' published partial
// tiles and folds them in FIXED order: every launch is bitwise reproducible
// (reference test_chfsi.py:234-241) and no SM idles in a wave tail, whatever
// (n, w) the locking leaves. A CTA computes and publishes its partial
// head-of-tile segment first, so owners never wait on a chain of peers.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <cstdlib>

#include "chfsi_internal.h"
#include "common.cuh"

// The kernel template and its launch descriptor are shared by the two
// translation units that instantiate it: cheb_step.cu (4M: four real DMMAs
// per complex block) and cheb_step_3m.cu (3M / Gauss: three).
namespace chfsi {
namespace k1 {

constexpr int BK = 16;             // complex elements per K slab (two 128-byte halves)
constexpr int HALF = 128;          // bytes per row per half-slab (one TMA box row)
constexpr int kMaxThreads = 512;
constexpr int kSlotDoubles = 8192; // partial-tile slot per CTA: ACC * THREADS <= this
constexpr int kMaxPeers = 7;       // fused all-gather: up to 8 ranks

struct StepParams {
  const double2* ycur;  // rows of Ycur matching the output rows (epilogue c*Ycur term)
  long long ldc;
  const double2* yprev;
  long long ldp;
  double2* ynext;
  long long ldn;
  int n, w;            // contraction length (== rows of H), columns of Y
  int m;               // output rows computed by this launch (row shard of H)
  int kblk_slabs;      // > 0: B operand in rank-blocked layout, K slabs per block
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
  unsigned* ticket;    // CTA ticket counter (logical CTA id = ticket - ticket_base)
  unsigned ticket_base;
  int dbg;             // diagnostics (CHFSI_K1_DEBUG): 2 = whole tiles only, 8 = trace, 16 = reversed
  unsigned long long* trace;  // dbg & 8: per CTA [start, owner wait begin, wait end, end, smid]
  // fused all-gather (multi-GPU row shards): every Ynext element is also
  // stored at ynext + peer_shift[k] — the same location of the rank-blocked
  // buffer on peer k, mapped into this process (NVLink P2P stores)
  long long peer_shift[kMaxPeers];
  int npeer;
};

// ------------------------------------------------------------ PTX helpers ---
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, unsigned bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, unsigned bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// fragment row g of an 8-row group -> smem row inside the group. Rows g and
// g+1 (same LDS.128 phase) land 4 apart, i.e. in opposite 64-byte halves
// of the 128B-swizzled row, so the 8 lanes of a phase hit 32 distinct banks.
__device__ __forceinline__ int sigma(int g) { return ((g & 1) << 2) | (g >> 1); }

// First stream-K iteration of CTA c: even split. (Measured: the warp
// schedulers favour the older of two co-resident CTAs — the lower blockIdx
// finishes first on every SM, ~40 % earlier — but neither a blockIdx-weighted
// split (the SM pairing is not fixed) nor dynamically grabbed fixed-boundary
// slices (owner folds then wait on slices queued behind a CTA's current work)
// beat the even static split; oversubscribing the grid only helps n >= 4096.)
__device__ __forceinline__ int sk_begin(const StepParams& p, int c) {
  return (int)((long long)c * p.sk_iters / p.sk_ctas);
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
  const long long idx = (long long)col * p.ldn + row;
  const double2 v = make_double2(tr, ti);
  p.ynext[idx] = v;
  for (int k = 0; k < p.npeer; ++k) p.ynext[idx + p.peer_shift[k]] = v;  // P2P store to peer k
}

// GROUPS = 2: one CTA per SM holds two 8-warp groups on the SAME tile that
// take alternate k-slabs (each group its own TMA producer and half of the
// stage ring) and add their partial tiles in fixed order at every segment
// end — 16 warps per SM without the priority imbalance of two co-resident
// CTAs (the older CTA's warps win the schedulers; measured ~40 % earlier).
//
// GAUSS: the 3M complex product. Per complex 8x8x4 block T1 += Ar*Br,
// T2 += Ai*Bi, T3 += (Ar +- Ai)*(Br + Bi) — three real DMMAs instead of four;
// the operand sums are one DADD per fragment (FP64 pipe, shared with DMMA:
// 12 DMMA + 4 DADD cost 1.05x 12 DMMA, tools/microbench/fp64_mix.cu). At the
// end of every tile segment the accumulators become Cr = T1 -+ T2,
// Ci = T3 - T1 -+ T2 (+ for conj(H)), so partial tiles, the fold and the
// epilogue are the same as for the 4M product. Work per complex MAC: 6 real
// flops executed (the 8-flop algorithmic count stays the metric).
//
// NH: 128-byte halves per k-slab (2: 16 complex, 4: 32 complex) — a deeper
// slab halves the per-slab barrier / proxy-fence / refill overhead per DMMA.
template <int BM, int BN, int WM, int WN, int STAGES, int MINB, bool CONJ, int GROUPS, bool GAUSS,
          int NH = 2>
__global__ void __launch_bounds__(GROUPS* WM* WN * 32, MINB)
    cheb_step_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const StepParams p) {
  constexpr int NWARPS = WM * WN;          // warps per group (one tile's worth)
  constexpr int THREADS = NWARPS * 32;     // threads per group
  static_assert(GROUPS == 1 || (GROUPS == 2 && STAGES % 2 == 0), "two groups need an even ring");
  constexpr int TM = BM / WM, TN = BN / WN;
  constexpr int MI = TM / 8, NI = TN / 8;
  constexpr int ACC = MI * NI * 4;
  constexpr int A_BYTES = BM * HALF;  // one half-slab of A
  constexpr int B_BYTES = BN * HALF;
  constexpr int STAGE_BYTES = NH * (A_BYTES + B_BYTES);
  static_assert(NH == 2 || NH == 4, "k-slab of 2 or 4 halves");
  static_assert(THREADS <= kMaxThreads && ACC * THREADS <= kSlotDoubles, "workspace bound");
  static_assert(MI >= 1 && NI >= 1, "warp tile too small");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "128B swizzle needs 1024B-aligned boxes");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128B-swizzled TMA destinations must be 1024-byte aligned (offset kept
  // relative to the __shared__ array so loads stay LDS, not generic LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  const unsigned smem0 = smem_u32(smem);
  const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);

  const int lane = threadIdx.x & 31;
  const int group = GROUPS == 1 ? 0 : (int)threadIdx.x / THREADS;
  const int tid = (int)threadIdx.x - group * THREADS;  // thread index within the group
  const int warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / WN, wn = warp % WN;
  // group-local barrier (named barrier 2 for group 0 when two groups run)
  auto gsync = [&]() {
    if (GROUPS == 1) __syncthreads();
    else asm volatile("bar.sync 2, %0;\n" ::"n"(THREADS) : "memory");
  };
  const int G = gridDim.x;
  // Logical CTA id = dispatch order: thread 0 takes a ticket from a counter
  // (p.ticket_base = the tickets of all earlier launches on this workspace).
  // A stream-K owner waits only for LOWER logical ids, i.e. for CTAs that
  // were dispatched before it and so are resident or done — and every CTA
  // publishes its partial tile before it could wait on anything. The wait
  // is therefore deadlock-free whatever order the hardware dispatches
  // blockIdx in and whatever other grids share the SMs (the two-chain
  // filter, side-stream reductions); with blockIdx the same proof would
  // rest on in-order dispatch. Fold order is by logical id: still fixed, so
  // every launch stays bitwise reproducible. (Under PDL all CTAs of the
  // previous launch took their tickets before this grid could start.)
  __shared__ int s_cta;
  if (threadIdx.x == 0) s_cta = (int)(atomicAdd(p.ticket, 1u) - p.ticket_base);
  __syncthreads();
  const int cta = (p.dbg & 16) ? G - 1 - s_cta : s_cta;  // 16: reversed (diagnostic)
  const int kiters = p.kiters;

  // ---- this CTA's slice of the linearised iteration space (64-bit once)
  const int dp_iters = p.dp_waves * kiters;
  int sb = 0, se = 0;
  if (cta < p.sk_ctas) {
    sb = sk_begin(p, cta);
    se = sk_begin(p, cta + 1);
  }
  const int total = dp_iters + (se - sb);
  if (total == 0) return;
  const bool tr = (p.dbg & 8) && threadIdx.x == 0;
  // Local order: [publish] [data-parallel tiles] [middle] [owner tail].
  //   publish: the head of the last SK tile when the range ends inside it —
  //            done first, so peers' partials are ready early;
  //   middle:  whole SK tiles (epilogue directly);
  //   tail:    the end of the first SK tile when the range starts inside it
  //            — the CTA owns that tile and folds the peers' partials, so it
  //            comes last, after the peers had the most time to publish.
  int pub_start = se, tail_end = sb;
  if (se > sb) {
    if (se % kiters != 0) {
      const int head = ((se - 1) / kiters) * kiters;
      pub_start = head > sb ? head : sb;
    }
    if (sb % kiters != 0) {
      const int nb = (sb / kiters + 1) * kiters;
      tail_end = nb < se ? nb : se;
    }
    if (tail_end > pub_start) tail_end = sb;  // range inside one tile, not at its end: all publish
  }
  const int pub = se - pub_start;
  const int mid_start = tail_end > sb ? tail_end : sb;
  const int e1 = pub, e2 = e1 + dp_iters, e3 = e2 + (pub_start - mid_start);

  struct Cursor {
    int j, tile, kk, m0, n0;
  };
  auto set_tile = [&](Cursor& c, int tile, int kk) {
    c.tile = tile;
    c.kk = kk;
    c.m0 = (tile / p.tiles_n) * BM;
    c.n0 = (tile % p.tiles_n) * BN;
  };
  auto set_sk = [&](Cursor& c, int it) { set_tile(c, p.sk_first + it / kiters, it % kiters); };
  auto enter = [&](Cursor& c) {  // first iteration of the phase holding c.j
    if (c.j < e1) set_sk(c, pub_start + c.j);
    else if (c.j < e2) set_tile(c, cta, 0);
    else if (c.j < e3) set_sk(c, mid_start + (c.j - e2));
    else set_sk(c, sb + (c.j - e3));
  };
  auto start = [&](Cursor& c) {
    c.j = 0;
    enter(c);
  };
  auto advance = [&](Cursor& c) {
    ++c.j;
    ++c.kk;
    if (c.j == e1 || c.j == e2 || c.j == e3) enter(c);
    else if (c.kk == kiters) set_tile(c, c.tile + ((c.j > e1 && c.j < e2) ? G : 1), 0);
  };
  // one elected thread: arm the stage's barrier and issue its TMA boxes
  // (what: 1 = the H panel, 2 = the Y panel, 3 = both; the barrier is armed
  // with the whole stage's bytes by whichever part comes first)
  auto issue = [&](const Cursor& c, int stage, int what = 3) {
    const unsigned dst = smem0 + stage * STAGE_BYTES, bar = full0 + 8 * stage;
    const int x = c.kk * (NH * BK);  // in doubles
    if (what & 1) {
      mbar_expect_tx(bar, STAGE_BYTES);
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) tma_load_2d(dst + hh * A_BYTES, &tmA, bar, x + hh * BK, c.m0);
    }
    if (!(what & 2)) return;
    if (p.kblk_slabs > 0) {  // rank-blocked Y: block q holds rows [q*kblk, (q+1)*kblk)
      const int q = c.kk / p.kblk_slabs, xl = (c.kk - q * p.kblk_slabs) * (NH * BK);
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
        tma_load_3d(dst + NH * A_BYTES + hh * B_BYTES, &tmB, bar, xl + hh * BK, c.n0, q);
    } else {
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
        tma_load_2d(dst + NH * A_BYTES + hh * B_BYTES, &tmB, bar, x + hh * BK, c.n0);
    }
  };

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, NWARPS);  // one arrival per warp of the consuming group
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // producer cursor (the group's thread 0): the group's iterations are
  // j = group, group + GROUPS, ... and stage j % STAGES is always its own
  Cursor lc;
  start(lc);
  for (int k = 0; k < group; ++k) advance(lc);
  // The H panels of the first ring stages are requested BEFORE the
  // dependency wait: H does not depend on the previous step (under PDL the
  // previous grid only writes Y and the stream-K scratch), so their HBM
  // latency overlaps the previous step's tail instead of opening every
  // launch with ~1 us of idle warps. The Y panels follow after the wait.
  if (tid == 0) {
    Cursor la = lc;
    for (int s = group; s < STAGES && la.j < total; s += GROUPS) {
      issue(la, s, 1);
      for (int k = 0; k < GROUPS; ++k) advance(la);
    }
  }
  // Programmatic dependent launch: the launch and the prologue above overlap
  // the previous step's tail; nothing the previous grid writes (Ycur, Yprev,
  // the stream-K partials and flags) is touched before this wait returns
  // (it returns at once when the launch had no programmatic dependency).
  // Dependents may be scheduled from here on: they wait the same way.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (tr) {
    p.trace[cta * 5 + 0] = gtimer();
    p.trace[cta * 5 + 4] = smid() | ((unsigned long long)blockIdx.x << 16);
  }
  if (tid == 0) {
    for (int s = group; s < STAGES && lc.j < total; s += GROUPS) {
      issue(lc, s, 2);
      for (int k = 0; k < GROUPS; ++k) advance(lc);
    }
  }

  // [.][.][0..1] real, [2..3] imag of C[g][2t+e] (GAUSS, inside a segment:
  // [0..1] T1, [2..3] T3, [4..5] T2)
  constexpr int NACC = GAUSS ? 6 : 4;
  double acc[MI][NI][NACC];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int e = 0; e < NACC; ++e) acc[i][j][e] = 0.0;

  const int sg = sigma(g);
  // Per 8-row block of the warp tile: ALL of its Ycur / Yprev reads first,
  // then the arithmetic and the stores. Ynext may alias Yprev, so the
  // compiler cannot move a later element's loads above an earlier element's
  // store: element by element, the epilogue was a chain of 2 * MI * NI
  // dependent L2 round trips per thread (ncu: 12 % long-scoreboard stalls).
  // Each thread still reads an element before it overwrites it, and no two
  // threads share an element. Same operation order as epilogue_store.
  // (Two row blocks per batch: 260 bytes of spills in the 255-register
  // variants, 2048x160 36.6 -> 35.7 TFLOP/s — one block per batch stays.)
  // (64-row tiles only — the n <= 4096 regime, where the epilogue is several
  // per cent of a launch; the 128-row tiles of the large shapes measured
  // 1-2 % slower with it: 5000x600 39.6 -> 39.1, 12000x1400 42.1 -> 41.3.)
  auto epilogue = [&](const Cursor& c) {
    if constexpr (BM != 64) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = c.m0 + wm * TM + i * 8 + sg;
            const int col = c.n0 + wn * TN + j * 8 + sigma(2 * t + e);
            if (row < p.m && col < p.w) epilogue_store(p, row, col, acc[i][j][e], acc[i][j][2 + e]);
          }
      return;
    }
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = c.m0 + wm * TM + i * 8 + sg;
      double2 yc[NI][2], yp[NI][2];
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = c.n0 + wn * TN + j * 8 + sigma(2 * t + e);
          const bool ok = row < p.m && col < p.w;
          yc[j][e] = (ok && p.read_cur) ? p.ycur[(long long)col * p.ldc + row] : make_double2(0.0, 0.0);
          yp[j][e] = (ok && p.read_prev) ? p.yprev[(long long)col * p.ldp + row] : make_double2(0.0, 0.0);
        }
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = c.n0 + wn * TN + j * 8 + sigma(2 * t + e);
          if (!(row < p.m && col < p.w)) continue;
          double tr = acc[i][j][e], ti = acc[i][j][2 + e];
          if (p.read_cur) {
            tr = dsub(tr, dmul(p.c, yc[j][e].x));
            ti = dsub(ti, dmul(p.c, yc[j][e].y));
          }
          tr = dmul(p.alpha, tr);
          ti = dmul(p.alpha, ti);
          if (p.read_prev) {
            tr = dsub(tr, dmul(p.beta, yp[j][e].x));
            ti = dsub(ti, dmul(p.beta, yp[j][e].y));
          }
          const long long idx = (long long)col * p.ldn + row;
          const double2 v = make_double2(tr, ti);
          p.ynext[idx] = v;
          for (int k = 0; k < p.npeer; ++k) p.ynext[idx + p.peer_shift[k]] = v;  // P2P store to peer k
        }
    }
  };

  // per-thread fragment byte offsets: row (warp base + sigma(g)) * 128, and
  // the swizzled chunk for even / odd k4 within a 128-byte half
  const int lo = (t ^ (g >> 1)) << 4;
  const int off_even = ((g & 1) << 6) | lo, off_odd = (((g & 1) ^ 1) << 6) | lo;
  const unsigned char* a_base = smem + (wm * TM + sg) * HALF;
  const unsigned char* b_base = smem + NH * A_BYTES + (wn * TN + sg) * HALF;
  // two groups: hand-over buffer for group 1's partial tile
  double* cbuf = reinterpret_cast<double*>(bars + 2 * STAGES);

  Cursor cc;
  start(cc);
  for (int j = 0; j < total; ++j) {
    const int stage = j % STAGES;
    const unsigned phase = (unsigned)(j / STAGES) & 1u;
    if (GROUPS == 1 || (j % GROUPS) == group) {
      mbar_wait(full0 + 8 * stage, phase);
      // mma.sync.aligned needs the whole warp converged: lane 0 of warp 0 may
      // still be issuing TMA (prologue) or spinning on an empty barrier
      __syncwarp();
      const unsigned char* sa = a_base + stage * STAGE_BYTES;
      const unsigned char* sbm = b_base + stage * STAGE_BYTES;
#pragma unroll
      for (int k4 = 0; k4 < NH * 2; ++k4) {
        const int off = (k4 & 1) ? off_odd : off_even;
        const unsigned char* ah = sa + (k4 >> 1) * A_BYTES + off;
        const unsigned char* bh = sbm + (k4 >> 1) * B_BYTES + off;
        double2 a[MI], b[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i) a[i] = lds128(ah + i * 8 * HALF);
#pragma unroll
        for (int jj = 0; jj < NI; ++jj) b[jj] = lds128(bh + jj * 8 * HALF);
        if constexpr (GAUSS) {
          double as[MI], bs[NI];
#pragma unroll
          for (int i = 0; i < MI; ++i) as[i] = CONJ ? dsub(a[i].x, a[i].y) : dadd(a[i].x, a[i].y);
#pragma unroll
          for (int jj = 0; jj < NI; ++jj) bs[jj] = dadd(b[jj].x, b[jj].y);
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int jj = 0; jj < NI; ++jj) {
              double(&t1)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][0]);
              double(&t3)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][2]);
              double(&t2)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][NACC - 2]);
              dmma884(t1, a[i].x, b[jj].x);
              dmma884(t2, a[i].y, b[jj].y);
              dmma884(t3, as[i], bs[jj]);
            }
          continue;
        }
        // Re/Im of (a or conj(a)) * b: four real DMMAs per complex 8x8x4 block
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < NI; ++jj) {
            double(&cr)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][0]);
            double(&ci)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][2]);
            dmma884(cr, a[i].x, b[jj].x);
            dmma884(ci, a[i].x, b[jj].y);
          }
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const double ai = a[i].y, nai = -a[i].y;
#pragma unroll
          for (int jj = 0; jj < NI; ++jj) {
            double(&cr)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][0]);
            double(&ci)[2] = *reinterpret_cast<double(*)[2]>(&acc[i][jj][2]);
            dmma884(cr, CONJ ? ai : nai, b[jj].y);
            dmma884(ci, CONJ ? nai : ai, b[jj].x);
          }
        }
      }
      // Release the stage; the group's elected thread refills it once every
      // warp of the group has. The fragments were read through the generic
      // proxy (LDS) and the refill is an async-proxy (TMA) write of the same
      // bytes: the proxy fence makes the reads complete before the release
      // (without it ptxas schedules the arrive ahead of the last LDS and a
      // slow warp can read refilled data). (Measured alternative: the
      // last-arriving warp refills via a shared counter — no empty-barrier
      // wait, but ~3 % slower at 2 CTAs/SM.)
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * stage);
      if (tid == 0 && lc.j < total) {
        mbar_wait(empty0 + 8 * stage, phase);
        issue(lc, stage);
        for (int k = 0; k < GROUPS; ++k) advance(lc);
      }
      // warp 0 must reconverge before its next mma.sync.aligned (lane 0 may
      // have spun on the empty barrier while lanes 1-31 ran ahead)
      __syncwarp();
    }

    // ---- end of a tile segment?
    const bool tile_end = cc.kk == kiters - 1;
    const bool pub_end = pub > 0 && j == pub - 1;
    if (tile_end || pub_end) {
      if constexpr (GAUSS) {  // (T1, T3, T2) -> (Cr, Ci)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < NI; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const double t1 = acc[i][jj][e], t3 = acc[i][jj][2 + e], t2 = acc[i][jj][NACC - 2 + e];
              acc[i][jj][e] = CONJ ? dadd(t1, t2) : dsub(t1, t2);
              acc[i][jj][2 + e] = CONJ ? dadd(dsub(t3, t1), t2) : dsub(dsub(t3, t1), t2);
              acc[i][jj][NACC - 2 + e] = 0.0;
            }
      }
      if (GROUPS == 2) {
        // group 1 hands its partial tile to group 0 (fixed order: group 0's
        // own slabs first, then group 1's)
        double* cb = cbuf + tid;
        if (group == 1) {
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int jj = 0; jj < NI; ++jj)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                cb[((i * NI + jj) * 4 + e) * THREADS] = acc[i][jj][e];
                acc[i][jj][e] = 0.0;
              }
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(2 * THREADS) : "memory");
        if (group == 0) {
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int jj = 0; jj < NI; ++jj)
#pragma unroll
              for (int e = 0; e < 4; ++e)
                acc[i][jj][e] = dadd(acc[i][jj][e], cb[((i * NI + jj) * 4 + e) * THREADS]);
        }
        // group 1 may refill the buffer only after group 0 has read it
        asm volatile("bar.sync 3, %0;\n" ::"n"(2 * THREADS) : "memory");
        if (group == 1) {
          advance(cc);
          continue;  // group 0 finishes the segment
        }
      }
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
        gsync();
        if (tid == 0) st_release(p.flags + cta, p.epoch);
      } else if (j < pub + dp_iters) {
        epilogue(cc);
      } else {
        const int tile_s0 = (cc.tile - p.sk_first) * kiters;  // first SK iteration of the tile
        if (tile_s0 >= sb) {
          epilogue(cc);
        } else {
          // owner: the peers are the CTAs whose ranges hold [tile_s0, sb)
          const int first =  // the CTA holding iteration tile_s0
              (int)(((long long)(tile_s0 + 1) * p.sk_ctas + p.sk_iters - 1) / p.sk_iters) - 1;
          if (tid == 0) {
            if (tr) p.trace[cta * 5 + 1] = gtimer();
            for (int q = first; q < cta; ++q)
              while (ld_acquire(p.flags + q) != p.epoch) __nanosleep(64);
            if (tr) p.trace[cta * 5 + 2] = gtimer();
          }
          gsync();
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
          for (int e = 0; e < NACC; ++e) acc[i][jj][e] = 0.0;
    }
    advance(cc);
  }
  if (tr) p.trace[cta * 5 + 3] = gtimer();
}

struct Variant {
  const void* fn;
  int bm, bn, groups, threads, smem;
  int nh;        // 128-byte halves per k-slab: the slab is 8*nh complex deep
  int resident;  // CTAs per SM actually achievable
};

template <int BM, int BN, int WM, int WN, int STAGES, int MINB, bool CONJ, int GROUPS, bool GAUSS,
          int NH = 2>
Variant make_variant() {
  Variant v{};
  auto fn = cheb_step_kernel<BM, BN, WM, WN, STAGES, MINB, CONJ, GROUPS, GAUSS, NH>;
  v.nh = NH;
  v.fn = reinterpret_cast<const void*>(fn);
  v.bm = BM;
  v.bn = BN;
  v.groups = GROUPS;
  v.threads = GROUPS * WM * WN * 32;
  constexpr int ACC = (BM / WM / 8) * (BN / WN / 8) * 4;
  v.smem = STAGES * NH * (BM + BN) * HALF + 2 * STAGES * 8 + 1024 +
           (GROUPS == 2 ? ACC * WM * WN * 32 * 8 : 0);  // + group hand-over buffer
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v.smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, v.threads, v.smem);
  v.resident = occ > 0 ? occ : 1;
  return v;
}

}  // namespace k1
}  // namespace chfsi
