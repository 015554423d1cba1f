// K1 host side: tiling choice, TMA descriptors, the persistent stream-K
// schedule and the launch (kernel template in cheb_step_kernel.cuh).
#include "cheb_step_kernel.cuh"

namespace chfsi {

namespace k1 {
const Variant* variant_3m(int bm, int bn, int groups, int warps, bool conj);  // cheb_step_3m.cu
const Variant* variant_3m_deep(int bm, int bn, int groups, int warps, bool conj);
}  // namespace k1

namespace {

using namespace k1;

// --------------------------------------------------------------- host ---

unsigned long long* g_trace = nullptr;  // CHFSI_K1_DEBUG & 8: last launch's per-CTA trace
int g_trace_grid = 0;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// 2-D map over a complex128 matrix seen as doubles: dim0 = 2*len (contiguous),
// dim1 = count vectors `ld` complex apart; box = 16 doubles x rows, 128B swizzle.
bool encode_map(CUtensorMap* map, const void* base, long long len, long long count, long long ld,
                int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)(2 * len), (cuuint64_t)count};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 16)};
  const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D map over the rank-blocked layout: block q, column j, row r at
// base + (q*count + j)*len + r (complex); box = 16 doubles x rows x 1.
bool encode_map_blocked(CUtensorMap* map, const void* base, long long len, long long count,
                        long long blocks, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * len), (cuuint64_t)count, (cuuint64_t)blocks};
  const cuuint64_t strides[2] = {(cuuint64_t)(len * 16), (cuuint64_t)(len * count * 16)};
  const cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// (bm, bn, groups) -> kernel configuration. Function-local statics: built
// once, on first use (the caller has set the device). 4M product here; the
// 3M registry lives in cheb_step_3m.cu (its own translation unit: the two
// sets compile in parallel).
const Variant* variant_4m(int bm, int bn, int groups, int warps, bool conj) {
#define CHFSI_V(BM_, BN_, WM_, WN_, ST_, MB_, GR_)                                               \
  if (bm == BM_ && bn == BN_ && groups == GR_ && (warps == 0 || warps == WM_ * WN_)) {           \
    static const Variant a = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, false, GR_, false>();    \
    static const Variant b = make_variant<BM_, BN_, WM_, WN_, ST_, MB_, true, GR_, false>();     \
    return conj ? &b : &a;                                                                       \
  }
  CHFSI_V(64, 16, 8, 1, 4, 2, 1)
  CHFSI_V(64, 32, 4, 2, 4, 2, 1)
  CHFSI_V(64, 64, 4, 2, 3, 2, 1)
  CHFSI_V(32, 32, 2, 2, 4, 3, 1)
  CHFSI_V(32, 64, 2, 2, 3, 3, 1)
  CHFSI_V(128, 32, 8, 2, 5, 1, 1)
  CHFSI_V(128, 16, 8, 1, 6, 1, 1)
  // two 8-warp groups per CTA, one CTA per SM (alternate k-slabs)
  CHFSI_V(64, 16, 8, 1, 10, 1, 2)
  CHFSI_V(64, 32, 4, 2, 8, 1, 2)
#undef CHFSI_V
  return nullptr;
}

// Complex product formulation of the K1 MMA loop: 3 = Gauss/3M (three real
// DMMAs per complex 8x8x4 block, operand sums on the FP64 pipe), 4 = four
// real DMMAs. Process-wide default from CHFSI_K1_PRODUCT (3 unless set to 4);
// chfsi_set_complex_product() overrides it (tests, tuning).
int g_product = [] {
  const char* e = getenv("CHFSI_K1_PRODUCT");
  return (e && atoi(e) == 4) ? 4 : 3;
}();

// k-slab depth preference of the 3M kernels: 2 (16 complex) or 4 (32
// complex) 128-byte halves; CHFSI_K1_NH or chfsi_set_k1_slab(). Deep-slab
// variants exist for the default 3M tiles; others keep 16-deep slabs.
// Measured (profiles/r02n_k1_slab_depth.txt, TFLOP/s at 8 flops/CMAC, 16 vs
// 32 deep): 2048x160 34.6 -> 35.9, 2048x100 27.8 -> 29.6, 2048x40 22.9 ->
// 24.6, 5000x600 39.0 -> 39.6, 12000x1400 41.5 -> 42.1; C2 sequence
// 306-311 -> 299 ms. Default 4 (CHFSI_K1_NH=2 restores 16-deep slabs).
int g_nh = [] {
  const char* e = getenv("CHFSI_K1_NH");
  return (e && atoi(e) == 2) ? 2 : 4;
}();

const Variant* variant(int bm, int bn, int groups, int warps, bool conj, int product,
                       bool allow_deep = true) {
  if (product == 0) product = g_product;
  if (product == 3 && g_nh == 4 && allow_deep) {
    if (const Variant* v = variant_3m_deep(bm, bn, groups, warps, conj)) return v;
  }
  if (product == 3) {
    if (const Variant* v = variant_3m(bm, bn, groups, warps, conj)) return v;
  }
  return variant_4m(bm, bn, groups, warps, conj);
}

}  // namespace

StepTiling choose_step_tiling(int n, int w) {
  if (g_product == 3) {
    // 3M product (profiles/r01_k1_3m_sweep.log, TFLOP/s at 8 flops per
    // complex MAC): the 3M kernels want 32x16 warp tiles with ~250 registers
    // (two warps per SM sub-partition) — 64x32 with 4 warps (2 CTAs/SM) or
    // 128x32 with 8 warps (1 CTA/SM): 2048x160 34.7, 4096x160 37.7,
    // 5000x600 39.0, 12000x1400 41.6; 64x16 with 4 warps when it pads
    // >10 % fewer columns (2048x100: 28.0 vs 26.5).
    // (round 2, 32-deep slabs, profiles/r03e_k1_narrow_tiles.txt, n = 2048:
    // 64x16 wins whenever it pads fewer columns — w = 144: 34.3 vs 32.8,
    // w = 80: 31.7 vs 27.8 — and at w <= 64 — w = 64: 30.5 vs 29.6; 64x32 at
    // equal padding above that — w = 96/128/160: 33.3/35.1/36.4 vs 32.4/33.6/34.0)
    const int p16 = ((w + 15) / 16) * 16, p32 = ((w + 31) / 32) * 32;
    StepTiling t{64, 32, 0};
    t.warps = 4;
    if (w <= 64 || p16 < p32) t.bn = 16;
    else if (n >= 8000 || w >= 400) {
      t.bm = 128;
      t.warps = 8;
    }
    return t;
  }
  // Measured on B200 (profiles/r01_k1_tiling.log, r01_k1_dual.log, TFLOP/s):
  //  * padding dominates at small w: 64x16 (8 warps x 8x16) runs at ~0.9x the
  //    speed of 64x32 per padded column, so it wins when it pads >10 % less;
  //  * n <= 3000: 64x32 with two CTAs per SM (29.3 at C2's 2048x160);
  //  * larger n: the two-group 64x32 CTA (one per SM, alternate k-slabs;
  //    no co-resident-CTA imbalance) gains 3-5 % (4096x160: 32.2 vs 30.7);
  //    the 16-warp 128x32 CTA is level with it once n >= 8000 or w >= 400
  //    (34.9 TFLOP/s = 94 % of the DMMA peak at C4).
  if (w <= 16) return StepTiling{64, 16, 0};
  const int pad16 = ((w + 15) / 16) * 16, pad32 = ((w + 31) / 32) * 32;
  if (pad16 * 10 < pad32 * 9) return StepTiling{64, 16, 0};
  if (n <= 3000) return StepTiling{64, 32, 0};
  if (n >= 8000 || w >= 400) return StepTiling{128, 32, 0};
  return StepTiling{64, 32, 0, 2};
}

int step_trace_copy(unsigned long long* host, int max_ctas) {
  if (!g_trace) return 0;
  const int n = g_trace_grid < max_ctas ? g_trace_grid : max_ctas;
  if (cudaMemcpy(host, g_trace, (size_t)n * 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return -1;
  return n;
}

size_t step_workspace_doubles(int max_grid) { return (size_t)max_grid * kSlotDoubles; }

int step_grid_size(int bn, bool conj) {
  const Variant* v = variant(64, bn, 1, 0, conj, 0);
  return v ? v->resident * kNumSMs : 0;
}

cudaError_t cheb_step_launch(const double2* h, long long ldh, bool conj_h, const double2* ycur,
                             long long ldc, const double2* yprev, long long ldp, double2* ynext,
                             long long ldn, int n, int w, double alpha, double c, double beta,
                             StepTiling tiling, const StepWorkspace& ws, cudaStream_t stream,
                             bool pdl) {
  const RowShard whole{n, 0, 0, nullptr, 0};
  return cheb_step_rows_launch(h, ldh, conj_h, ycur, ldc, yprev, ldp, ynext, ldn, n, w, alpha, c,
                               beta, whole, tiling, ws, stream, nullptr, 0, pdl);
}

cudaError_t cheb_step_rows_launch(const double2* h, long long ldh, bool conj_h, const double2* ycur,
                                  long long ldc, const double2* yprev, long long ldp, double2* ynext,
                                  long long ldn, int n, int w, double alpha, double c, double beta,
                                  const RowShard& shard, StepTiling tiling, const StepWorkspace& ws,
                                  cudaStream_t stream, const long long* peer_shift, int npeer,
                                  bool pdl) {
  if (npeer < 0 || npeer > kMaxPeers) return cudaErrorInvalidValue;
  const int m = shard.rows;
  if (n <= 0 || w <= 0 || m <= 0) return cudaSuccess;
  if (tiling.bm == 0) tiling = choose_step_tiling(n, w);
  // a rank-blocked operand needs whole slabs per rank block
  const bool deep_ok = shard.kblk <= 0 || shard.kblk % 32 == 0;
  const Variant* vp =
      variant(tiling.bm, tiling.bn, tiling.groups ? tiling.groups : 1, tiling.warps, conj_h,
              tiling.product, deep_ok);
  if (vp == nullptr) return cudaErrorInvalidValue;
  const Variant& v = *vp;
  int grid = v.resident * kNumSMs;
  if (tiling.split > 0 && tiling.split < grid) grid = tiling.split;  // test/tuning override
  if (grid > ws.max_grid) return cudaErrorInvalidValue;

  // A: the shard's rows of H (m rows, contraction n). B: Ycur, either plain
  // column-major (ld ldc) or rank-blocked (kblk rows per block, nblk blocks).
  alignas(64) CUtensorMap tmA, tmB;
  const bool blocked = shard.kblk > 0;
  const int slab = 8 * v.nh;  // complex elements per k-slab
  if (blocked && (shard.kblk % slab != 0 || (long long)shard.kblk * shard.nblk < n))
    return cudaErrorInvalidValue;
  if (!encode_map(&tmA, h, n, m, ldh, v.bm)) return cudaErrorInvalidValue;
  if (blocked ? !encode_map_blocked(&tmB, ycur, shard.kblk, w, shard.nblk, v.bn)
              : !encode_map(&tmB, ycur, n, w, ldc, v.bn))
    return cudaErrorInvalidValue;

  StepParams p{};
  p.ycur = shard.ycur_rows ? shard.ycur_rows : ycur;
  p.ldc = shard.ycur_rows ? shard.ldcr : ldc;
  p.m = m;
  p.kblk_slabs = blocked ? shard.kblk / slab : 0;
  p.yprev = yprev ? yprev : ynext;
  p.ldp = yprev ? ldp : ldn;
  p.ynext = ynext;
  p.ldn = ldn;
  p.npeer = npeer;
  for (int k = 0; k < npeer; ++k) p.peer_shift[k] = peer_shift[k];
  p.n = n;
  p.w = w;
  p.tiles_n = (w + v.bn - 1) / v.bn;
  const int tiles_m = (m + v.bm - 1) / v.bm;
  const long long tiles = (long long)tiles_m * p.tiles_n;
  p.kiters = blocked ? shard.nblk * (shard.kblk / slab) : (n + slab - 1) / slab;
  static const int dbg = [] {
    const char* e = getenv("CHFSI_K1_DEBUG");
    return e ? atoi(e) : 0;
  }();
  p.dbg = dbg;
  if (dbg & 8) {
    static unsigned long long* trace_buf = nullptr;
    if (!trace_buf && cudaMalloc(&trace_buf, 4096 * 5 * sizeof(unsigned long long)) != cudaSuccess)
      return cudaErrorMemoryAllocation;
    g_trace = trace_buf;
    g_trace_grid = grid;
    cudaMemsetAsync(trace_buf, 0, (size_t)grid * 5 * sizeof(unsigned long long), stream);
    p.trace = trace_buf;
  }
  if ((dbg & 2) && tiles <= grid) grid = (int)tiles;  // one whole tile per CTA, no stream-K
  p.dp_waves = tiles >= 2LL * grid ? (int)(tiles / grid) - 1 : 0;
  if ((dbg & 2) && tiles == grid) p.dp_waves = 1;
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
  p.ticket = ws.flags + ws.max_grid;  // every CTA of this launch takes one ticket
  p.ticket_base = *ws.tickets;
  *ws.tickets += (unsigned)grid;
  void* args[] = {&tmA, &tmB, &p};
  note_launch();
  // Programmatic dependent launch between consecutive steps of one filter
  // chain (the kernel waits on griddepcontrol before touching the previous
  // step's outputs). Only there: a PDL launch after other work let K1 CTAs
  // park on SM slots early and cost 8 % at C2. CHFSI_K1_PDL=0 disables it.
  static const bool pdl_env = [] {
    const char* e = getenv("CHFSI_K1_PDL");
    return !(e && atoi(e) == 0);
  }();
  pdl = pdl && pdl_env;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(v.threads);
  cfg.dynamicSmemBytes = v.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, v.fn, args);
}

int set_complex_product(int product) {
  if (product != 3 && product != 4) return -1;
  const int old = g_product;
  g_product = product;
  return old;
}

int complex_product() { return g_product; }

int set_k1_slab(int nh) {
  if (nh != 2 && nh != 4) return -1;
  const int old = g_nh;
  g_nh = nh;
  return old;
}

}  // namespace chfsi
