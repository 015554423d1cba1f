// C-ABI of libchfsi (declared in include/chfsi.h): context management,
// cuBLAS/cuSOLVER calls for the small dense factorizations, and the
// orchestration of the hand-written kernels (cheb_step.cu, aux_kernels.cu).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "abi_internal.h"

using chfsi::LanczosState;

namespace chfsi {
static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace chfsi

namespace chfsi {
static thread_local std::string g_last_error;
// Cholesky-QR2 panel kernels (panel_kernels.cu) on/off: CHFSI_PANEL_KERNELS, chfsi_set_panel_kernels()
static std::atomic<bool> g_panel_kernels{[] {
  const char* e = getenv("CHFSI_PANEL_KERNELS");
  return !(e && atoi(e) == 0);
}()};
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int ensure_pinned(chfsi_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->pinned_bytes) return CHFSI_OK;
  CK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->pinned) CK_CUDA(cudaFreeHost(ctx->pinned));
  ctx->pinned = nullptr;
  ctx->pinned_bytes = 0;
  bytes = std::max<size_t>(bytes, 4096);
  CK_CUDA(cudaMallocHost(&ctx->pinned, bytes));
  ctx->pinned_bytes = bytes;
  return CHFSI_OK;
}
}  // namespace chfsi

namespace {

using chfsi::fail;

int ensure_ws(chfsi_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return CHFSI_OK;
  CK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->ws) CK_CUDA(cudaFree(ctx->ws));
  ctx->ws = nullptr;
  ctx->ws_bytes = 0;
  CK_CUDA(cudaMalloc(&ctx->ws, bytes));
  ctx->ws_bytes = bytes;
  return CHFSI_OK;
}

int ensure_scratch(chfsi_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes) return CHFSI_OK;
  CK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->scratch) CK_CUDA(cudaFree(ctx->scratch));
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  CK_CUDA(cudaMalloc(&ctx->scratch, bytes));
  ctx->scratch_bytes = bytes;
  return CHFSI_OK;
}

cublasOperation_t op_of(char t) {
  switch (t) {
    case 'T': case 't': return CUBLAS_OP_T;
    case 'C': case 'c': return CUBLAS_OP_C;
    default: return CUBLAS_OP_N;
  }
}

bool valid_op(char t) { return t == 'N' || t == 'n' || t == 'T' || t == 't' || t == 'C' || t == 'c'; }

}  // namespace

extern "C" {

int chfsi_version(void) { return 1; }

long long chfsi_launch_count(void) { return chfsi::g_launches.load(std::memory_order_relaxed); }

const char* chfsi_last_error(void) { return chfsi::g_last_error.c_str(); }

int chfsi_ctx_create(int device, chfsi_ctx** out) {
  CK_ARG(out != nullptr, "out is NULL");
  *out = nullptr;
  CK_CUDA(cudaSetDevice(device));
  chfsi_ctx* ctx = new chfsi_ctx();
  ctx->device = device;
  if (cublasCreate(&ctx->blas) != CUBLAS_STATUS_SUCCESS) {
    delete ctx;
    return fail(CHFSI_ECUBLAS, "cublasCreate failed");
  }
  if (cusolverDnCreate(&ctx->solver) != CUSOLVER_STATUS_SUCCESS) {
    cublasDestroy(ctx->blas);
    delete ctx;
    return fail(CHFSI_ECUSOLVER, "cusolverDnCreate failed");
  }
  // deterministic, exact FP64 arithmetic in the library GEMMs
  cublasSetAtomicsMode(ctx->blas, CUBLAS_ATOMICS_NOT_ALLOWED);
  cublasSetMathMode(ctx->blas, CUBLAS_DEFAULT_MATH);
  cublasSetPointerMode(ctx->blas, CUBLAS_POINTER_MODE_HOST);
  CK_CUDA(cudaMalloc(&ctx->partial, chfsi::kRedBlocks * sizeof(double)));
  CK_CUDA(cudaMalloc(&ctx->scalars, 16 * sizeof(double)));
  CK_CUDA(cudaMalloc(&ctx->dinfo, 4 * sizeof(int)));
  CK_CUDA(cudaMalloc(&ctx->lstate, sizeof(LanczosState)));
  CK_CUDA(cudaMalloc(&ctx->red_counter, sizeof(unsigned)));
  CK_CUDA(cudaMemset(ctx->red_counter, 0, sizeof(unsigned)));
  // K1 stream-K scratch: partial tiles and ready flags for every resident CTA
  ctx->step_ws.max_grid = chfsi::kNumSMs * 4;
  CK_CUDA(cudaMalloc(&ctx->step_ws.partials,
                     chfsi::step_workspace_doubles(ctx->step_ws.max_grid) * sizeof(double)));
  CK_CUDA(cudaMalloc(&ctx->step_ws.flags, (ctx->step_ws.max_grid + 1) * sizeof(unsigned)));
  CK_CUDA(cudaMemset(ctx->step_ws.flags, 0, (ctx->step_ws.max_grid + 1) * sizeof(unsigned)));
  ctx->step_ws.epoch = &ctx->step_epoch;
  ctx->step_ws.tickets = &ctx->step_tickets;
  *out = ctx;
  return CHFSI_OK;
}

int chfsi_ctx_destroy(chfsi_ctx* ctx) {
  if (!ctx) return CHFSI_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  cudaDeviceSynchronize();
  if (ctx->blas) cublasDestroy(ctx->blas);
  if (ctx->solver) cusolverDnDestroy(ctx->solver);
  cudaFree(ctx->ws);
  cudaFree(ctx->scratch);
  cudaFree(ctx->eig_ws);
  cudaFree(ctx->partial);
  cudaFree(ctx->scalars);
  cudaFree(ctx->dinfo);
  cudaFree(ctx->lstate);
  cudaFree(ctx->panel_linv);
  cudaFree(ctx->red_counter);
  cudaFree(ctx->step_ws.partials);
  cudaFree(ctx->step_ws.flags);
  if (ctx->aux_stream) {
    cudaStreamSynchronize(ctx->aux_stream);
    cudaStreamDestroy(ctx->aux_stream);
    cudaEventDestroy(ctx->fork_ev);
    cudaEventDestroy(ctx->join_ev);
    cudaFree(ctx->step_ws2.partials);
    cudaFree(ctx->step_ws2.flags);
  }
  for (cudaEvent_t e : ctx->loop_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->qr_pinned) cudaFreeHost(ctx->qr_pinned);
  if (ctx->nd_pinned) cudaFreeHost(ctx->nd_pinned);
  delete ctx;
  return CHFSI_OK;
}

int chfsi_ctx_set_tiling(chfsi_ctx* ctx, int bm, int bn, int split) {
  CK_ARG(ctx, "ctx is NULL");
  if (bm == 0) {
    ctx->tiling = chfsi::StepTiling{0, 0, 0};
    return CHFSI_OK;
  }
  CK_ARG((bm == 32 || bm == 64 || bm == 128) && (bn == 16 || bn == 32 || bn == 64) && split >= 0 &&
             split <= ctx->step_ws.max_grid,
         "unsupported K1 tiling");
  ctx->tiling = chfsi::StepTiling{bm, bn, split};
  return CHFSI_OK;
}

int chfsi_ctx_set_filter_chains(chfsi_ctx* ctx, int chains) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(chains == 1 || chains == 2, "chains must be 1 or 2");
  ctx->filter_chains = chains;
  return CHFSI_OK;
}

int chfsi_ctx_set_step_groups(chfsi_ctx* ctx, int groups) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(groups == 1 || groups == 2, "groups must be 1 or 2");
  CK_ARG(ctx->tiling.bm != 0, "set a tiling first (chfsi_ctx_set_tiling)");
  CK_ARG(groups == 1 || (ctx->tiling.bm == 64 && (ctx->tiling.bn == 16 || ctx->tiling.bn == 32)),
         "two-group K1 exists for 64x16 and 64x32");
  ctx->tiling.groups = groups;
  return CHFSI_OK;
}

int chfsi_ctx_set_step_warps(chfsi_ctx* ctx, int warps) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(warps == 0 || warps == 4 || warps == 8 || warps == 16, "warps must be 0, 4, 8 or 16");
  CK_ARG(warps == 0 || ctx->tiling.bm != 0, "set a tiling first (chfsi_ctx_set_tiling)");
  ctx->tiling.warps = warps;
  return CHFSI_OK;
}

int chfsi_ctx_set_stream(chfsi_ctx* ctx, void* stream) {
  CK_ARG(ctx, "ctx is NULL");
  ctx->stream = static_cast<cudaStream_t>(stream);
  CK_BLAS(cublasSetStream(ctx->blas, ctx->stream));
  CK_SOLVER(cusolverDnSetStream(ctx->solver, ctx->stream));
  return CHFSI_OK;
}

// ------------------------------------------------------------------- K1 ---

int chfsi_cheb_step_z(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                      const void* ycur, long long ldc, const void* yprev, long long ldp,
                      void* ynext, long long ldn, double alpha, double c, double beta) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(n >= 0 && w >= 0, "negative size");
  if (n == 0 || w == 0) return CHFSI_OK;
  CK_ARG(H && ycur && ynext, "NULL operand");
  CK_ARG(ldh >= n && ldc >= n && ldn >= n && (!yprev || ldp >= n), "leading dimension < n");
  CK_ARG(ycur != ynext, "Ycur must not alias Ynext");
  CK_CUDA(chfsi::cheb_step_launch(static_cast<const double2*>(H), ldh, conj_h != 0,
                                  static_cast<const double2*>(ycur), ldc,
                                  static_cast<const double2*>(yprev), ldp,
                                  static_cast<double2*>(ynext), ldn, n, w, alpha, c, beta,
                                  ctx->tiling, ctx->step_ws, ctx->stream));
  return CHFSI_OK;
}

int chfsi_cheb_step_rows_z(chfsi_ctx* ctx, int n, int rows, int w, const void* H_rows, long long ldh,
                           int conj_h, const void* ycur, long long ldc, int kblk, int nblk,
                           const void* ycur_rows, long long ldcr, const void* yprev, long long ldp,
                           void* ynext, long long ldn, double alpha, double c, double beta) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(n >= 0 && rows >= 0 && w >= 0, "negative size");
  if (n == 0 || w == 0 || rows == 0) return CHFSI_OK;
  CK_ARG(H_rows && ycur && ynext && ycur_rows, "NULL operand");
  CK_ARG(ldh >= n && ldn >= rows && ldcr >= rows && (!yprev || ldp >= rows), "leading dimension");
  CK_ARG(kblk == 0 ? ldc >= n : (kblk % 16 == 0 && (long long)kblk * nblk >= n),
         "blocked layout needs kblk % 16 == 0 and kblk * nblk >= n");
  const chfsi::RowShard shard{rows, kblk, nblk, static_cast<const double2*>(ycur_rows), ldcr};
  CK_CUDA(chfsi::cheb_step_rows_launch(static_cast<const double2*>(H_rows), ldh, conj_h != 0,
                                       static_cast<const double2*>(ycur), ldc,
                                       static_cast<const double2*>(yprev), ldp,
                                       static_cast<double2*>(ynext), ldn, n, w, alpha, c, beta, shard,
                                       ctx->tiling.bm ? ctx->tiling : chfsi::choose_step_tiling(rows, w),
                                       ctx->step_ws, ctx->stream));
  return CHFSI_OK;
}

int chfsi_cheb_step_rows_peers_z(chfsi_ctx* ctx, int n, int rows, int w, const void* H_rows,
                                 long long ldh, int conj_h, const void* ycur, long long ldc, int kblk,
                                 int nblk, const void* ycur_rows, long long ldcr, const void* yprev,
                                 long long ldp, void* ynext, long long ldn, double alpha, double c,
                                 double beta, const void* const* peer_ynext, int npeer) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(n >= 0 && rows >= 0 && w >= 0, "negative size");
  if (n == 0 || w == 0 || rows == 0) return CHFSI_OK;
  CK_ARG(H_rows && ycur && ynext && ycur_rows, "NULL operand");
  CK_ARG(npeer >= 0 && npeer <= 7 && (npeer == 0 || peer_ynext), "0 <= npeer <= 7 peer outputs");
  long long shift[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < npeer; ++k) {
    const long long d = reinterpret_cast<const char*>(peer_ynext[k]) -
                        reinterpret_cast<const char*>(ynext);
    CK_ARG(peer_ynext[k] && d % (long long)sizeof(double2) == 0, "peer outputs must be 16-byte aligned");
    shift[k] = d / (long long)sizeof(double2);
  }
  CK_ARG(ldh >= n && ldn >= rows && ldcr >= rows && (!yprev || ldp >= rows), "leading dimension");
  CK_ARG(kblk == 0 ? ldc >= n : (kblk % 16 == 0 && (long long)kblk * nblk >= n),
         "blocked layout needs kblk % 16 == 0 and kblk * nblk >= n");
  const chfsi::RowShard shard{rows, kblk, nblk, static_cast<const double2*>(ycur_rows), ldcr};
  CK_CUDA(chfsi::cheb_step_rows_launch(static_cast<const double2*>(H_rows), ldh, conj_h != 0,
                                       static_cast<const double2*>(ycur), ldc,
                                       static_cast<const double2*>(yprev), ldp,
                                       static_cast<double2*>(ynext), ldn, n, w, alpha, c, beta, shard,
                                       ctx->tiling.bm ? ctx->tiling : chfsi::choose_step_tiling(rows, w),
                                       ctx->step_ws, ctx->stream, shift, npeer));
  return CHFSI_OK;
}

int chfsi_filter_degrees_z(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                           const void* y0, long long ldy0, void* buf_a, void* buf_b, long long ldb,
                           const int* degs, double a, double b, double scale_ref, void** result) {
  return chfsi::filter_degrees_impl(ctx, n, w, H, ldh, conj_h, y0, ldy0, nullptr, 0, buf_a, buf_b,
                                    ldb, degs, a, b, scale_ref, result);
}

}  // extern "C"

namespace chfsi {

int filter_degrees_impl(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                        const void* y0, long long ldy0, const void* hy0_, long long ldhy0,
                        void* buf_a, void* buf_b, long long ldb, const int* degs, double a, double b,
                        double scale_ref, void** result) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(n >= 0 && w >= 0, "negative size");
  CK_ARG(result, "result is NULL");
  CK_ARG(buf_a != buf_b && y0 != buf_a, "buffers must be distinct (y0 may equal buf_b)");
  CK_ARG(w == 0 || degs, "degs is NULL");
  for (int j = 0; j < w; ++j)
    CK_ARG(degs[j] >= 1 && (j == 0 || degs[j] >= degs[j - 1]),
           "per-column degrees must be >= 1 and non-decreasing");
  if (w == 0) {
    *result = buf_a;
    return CHFSI_OK;
  }
  const int dmax = degs[w - 1];
  std::vector<double> al(dmax), be(dmax);
  double c = 0.0;
  CK(chfsi_filter_coeffs(dmax, a, b, scale_ref, &c, al.data(), be.data()));
  *result = (dmax % 2) ? buf_a : buf_b;
  if (n == 0) return CHFSI_OK;
  // One recurrence for all columns (the step coefficients do not depend on
  // the final degree); step j only runs the columns whose degree exceeds j,
  // a suffix [first, w) because degrees are sorted.
  const double2* hh = static_cast<const double2*>(H);
  const double2* prev = nullptr;
  long long ldp = 0;
  const double2* cur = static_cast<const double2*>(y0);
  long long ldcur = ldy0;
  int first = 0;
  for (int j = 0; j < dmax; ++j) {
    while (first < w && degs[first] <= j) ++first;
    double2* dst = static_cast<double2*>((j % 2 == 0) ? buf_a : buf_b);
    const int wa = w - first;
    const chfsi::StepTiling tiling = ctx->tiling.bm ? ctx->tiling : chfsi::choose_step_tiling(n, wa);
    const double2* hy0 = static_cast<const double2*>(hy0_);
    if (j == 0 && hy0)  // H Y0 known: elementwise first step
      CK_CUDA(chfsi::cheb_first_step_launch(hy0 + first * ldhy0, ldhy0, cur + first * ldcur, ldcur,
                                            dst + first * ldb, ldb, n, wa, al[0], c, ctx->stream));
    else
      CK_CUDA(chfsi::cheb_step_launch(hh, ldh, conj_h != 0, cur + first * ldcur, ldcur,
                                      prev ? prev + first * ldp : nullptr, ldp, dst + first * ldb,
                                      ldb, n, wa, al[j], c, be[j], tiling, ctx->step_ws, ctx->stream,
                                      /*pdl=*/j > 1 || (j == 1 && !hy0)));
    prev = cur;
    ldp = ldcur;
    cur = dst;
    ldcur = ldb;
  }
  // a column of degree d ended in the buffer of step d-1 (buf_a when d is
  // odd): move the groups whose parity differs from dmax's into *result
  double2* res = static_cast<double2*>(*result);
  for (int j0 = 0; j0 < w;) {
    int j1 = j0;
    while (j1 < w && (degs[j1] % 2) == (degs[j0] % 2)) ++j1;
    if ((degs[j0] % 2) != (dmax % 2)) {
      const double2* src = static_cast<const double2*>((degs[j0] % 2) ? buf_a : buf_b);
      CK_CUDA(cudaMemcpy2DAsync(res + j0 * ldb, ldb * sizeof(double2), src + j0 * ldb,
                                ldb * sizeof(double2), (size_t)n * sizeof(double2), j1 - j0,
                                cudaMemcpyDeviceToDevice, ctx->stream));
    }
    j0 = j1;
  }
  return CHFSI_OK;
}

}  // namespace chfsi

extern "C" {

int chfsi_filter_coeffs(int deg, double a, double b, double scale_ref, double* c, double* alphas,
                        double* betas) {
  CK_ARG(deg >= 1, "polynomial degree must be >= 1");
  CK_ARG(c && alphas && betas, "NULL output");
  // chfsi.py:198-207, operation for operation
  const double e = (b - a) / 2;
  const double cc = (b + a) / 2;
  double sigma = e / (scale_ref - cc);
  const double tau = 2.0 / sigma;
  *c = cc;
  alphas[0] = sigma / e;
  betas[0] = 0.0;
  for (int j = 1; j < deg; ++j) {
    const double sigma_new = 1.0 / (tau - sigma);
    alphas[j] = 2 * sigma_new / e;
    betas[j] = sigma * sigma_new;
    sigma = sigma_new;
  }
  return CHFSI_OK;
}

namespace {

// deg recurrence steps over columns [c0, c0 + w) on `stream`
int filter_range(chfsi_ctx* ctx, cudaStream_t stream, const chfsi::StepWorkspace& ws,
                 chfsi::StepTiling tiling, int n, int c0, int w, const double2* hh, long long ldh,
                 bool conj, const double2* y0, long long ldy0, double2* buf_a, double2* buf_b,
                 long long ldb, int deg, const double* al, const double* be, double c,
                 const double2* hy0 = nullptr, long long ldhy0 = 0) {
  const double2* prev = nullptr;
  long long ldp = 0;
  const double2* cur = y0 + (long long)c0 * ldy0;
  long long ldcur = ldy0;
  for (int j = 0; j < deg; ++j) {
    double2* dst = ((j % 2 == 0) ? buf_a : buf_b) + (long long)c0 * ldb;
    if (j == 0 && hy0)  // H Y0 known (the previous Rayleigh-Ritz's rotated H P)
      CK_CUDA(chfsi::cheb_first_step_launch(hy0 + (long long)c0 * ldhy0, ldhy0, cur, ldcur, dst, ldb,
                                            n, w, al[0], c, stream));
    else
      CK_CUDA(chfsi::cheb_step_launch(hh, ldh, conj, cur, ldcur, prev, ldp, dst, ldb, n, w, al[j], c,
                                      be[j], tiling, ws, stream, /*pdl=*/j > 1 || (j == 1 && !hy0)));
    prev = cur;
    ldp = ldcur;
    cur = dst;
    ldcur = ldb;
  }
  return CHFSI_OK;
}

int ensure_aux_stream(chfsi_ctx* ctx) {
  if (ctx->aux_stream) return CHFSI_OK;
  // the second filter chain runs at the priority of the context's stream
  // (a high-priority solver stream must not lose half its filter to it)
  int prio = 0;
  CK_CUDA(cudaStreamGetPriority(ctx->stream, &prio));
  CK_CUDA(cudaStreamCreateWithPriority(&ctx->aux_stream, cudaStreamNonBlocking, prio));
  CK_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
  CK_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
  ctx->step_ws2.max_grid = ctx->step_ws.max_grid;
  CK_CUDA(cudaMalloc(&ctx->step_ws2.partials,
                     chfsi::step_workspace_doubles(ctx->step_ws2.max_grid) * sizeof(double)));
  CK_CUDA(cudaMalloc(&ctx->step_ws2.flags, (ctx->step_ws2.max_grid + 1) * sizeof(unsigned)));
  CK_CUDA(cudaMemset(ctx->step_ws2.flags, 0, (ctx->step_ws2.max_grid + 1) * sizeof(unsigned)));
  ctx->step_ws2.epoch = &ctx->step_epoch2;
  ctx->step_ws2.tickets = &ctx->step_tickets2;
  return CHFSI_OK;
}

}  // namespace

int chfsi_filter_z(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                   const void* y0, long long ldy0, void* buf_a, void* buf_b, long long ldb,
                   int deg, double a, double b, double scale_ref, void** result) {
  return chfsi::filter_z_impl(ctx, n, w, H, ldh, conj_h, y0, ldy0, nullptr, 0, buf_a, buf_b, ldb, deg,
                              a, b, scale_ref, result);
}

}  // extern "C"

namespace chfsi {

int filter_z_impl(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                  const void* y0, long long ldy0, const void* hy0_, long long ldhy0, void* buf_a,
                  void* buf_b, long long ldb, int deg, double a, double b, double scale_ref,
                  void** result) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(deg >= 1, "polynomial degree must be >= 1");
  CK_ARG(n >= 0 && w >= 0, "negative size");
  CK_ARG(result, "result is NULL");
  CK_ARG(buf_a != buf_b && y0 != buf_a, "buffers must be distinct (y0 may equal buf_b)");
  std::vector<double> al(deg), be(deg);
  double c = 0.0;
  CK(chfsi_filter_coeffs(deg, a, b, scale_ref, &c, al.data(), be.data()));
  *result = (deg % 2) ? buf_a : buf_b;
  if (n == 0 || w == 0) return CHFSI_OK;
  const double2* hh = static_cast<const double2*>(H);
  const double2* yy = static_cast<const double2*>(y0);
  double2* ba = static_cast<double2*>(buf_a);
  double2* bb = static_cast<double2*>(buf_b);
  const double2* hy0 = static_cast<const double2*>(hy0_);
  static const int env_chains = [] {
    const char* e = getenv("CHFSI_FILTER_STREAMS");  // 1 disables the two-chain filter
    return e ? atoi(e) : 2;
  }();
  const int streams = std::min(env_chains, ctx->filter_chains);
  // Columns are independent through the recurrence: two column halves run
  // as two concurrent launch chains (the context's stream and an auxiliary
  // one), one CTA per SM each. On every SM the warp schedulers favour the
  // older of two co-resident CTAs, which finishes ~40 % earlier; with two
  // chains the early CTA's SM slot starts its chain's next step instead of
  // idling (measured at n = 2048: w=160 29.2 -> 32.0 TFLOP/s, w=123
  // 27.5 -> 30.1, w=64 25.9 -> 28.5; n = 4096..8192 +2-5 % over the
  // one-CTA-per-SM tiles). Used for n < 10000 when the split is balanced
  // (w1 >= 0.6 w0, halves 32-aligned): a thin second chain (w=80 -> 64+16,
  // w=200 -> 128+72) loses to one chain.
  const int w0 = ((w / 2 + 31) / 32) * 32, w1 = w - w0;
  if (streams == 2 && ctx->tiling.bm == 0 && w1 > 0 && 10 * w1 >= 6 * w0) {
    // each chain: the 8-warp 64-row tile (64x16 when it pads >10 % less)
    auto chain_tiling = [](int wc) {
      const int p16 = ((wc + 15) / 16) * 16, p32 = ((wc + 31) / 32) * 32;
      chfsi::StepTiling t = p16 * 10 < p32 * 9 ? chfsi::StepTiling{64, 16, 0} : chfsi::StepTiling{64, 32, 0};
      if (chfsi::complex_product() == 3) t.warps = 4;  // the 3M kernels' 4-warp 64-row tiles
      return t;
    };
    chfsi::StepTiling t0 = chain_tiling(w0), t1 = chain_tiling(w1);
    // (n >= 10000: the single 16-warp 128x32 chain is ahead, 34.9 vs 34.2 at C4.
    // The 3M kernels — two warps per sub-partition, no co-resident-CTA
    // imbalance — gain from two chains only at C1-like sizes: 512x48 5.2 ->
    // 5.8, level at 2048x64..5000x250, behind at 2048x160 34.5 vs 32.2,
    // profiles/r01_k1_3m_sweep.log.)
    if (n < (chfsi::complex_product() == 3 ? 1500 : 10000)) {
      CK(ensure_aux_stream(ctx));
      t0.split = chfsi::kNumSMs;
      t1.split = chfsi::kNumSMs;
      CK_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
      CK_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->fork_ev, 0));
      CK(filter_range(ctx, ctx->stream, ctx->step_ws, t0, n, 0, w0, hh, ldh, conj_h != 0, yy, ldy0,
                      ba, bb, ldb, deg, al.data(), be.data(), c, hy0, ldhy0));
      CK(filter_range(ctx, ctx->aux_stream, ctx->step_ws2, t1, n, w0, w1, hh, ldh, conj_h != 0, yy,
                      ldy0, ba, bb, ldb, deg, al.data(), be.data(), c, hy0, ldhy0));
      CK_CUDA(cudaEventRecord(ctx->join_ev, ctx->aux_stream));
      CK_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
      return CHFSI_OK;
    }
  }
  const chfsi::StepTiling tiling =
      ctx->tiling.bm ? ctx->tiling : chfsi::choose_step_tiling(n, w);
  return filter_range(ctx, ctx->stream, ctx->step_ws, tiling, n, 0, w, hh, ldh, conj_h != 0, yy,
                      ldy0, ba, bb, ldb, deg, al.data(), be.data(), c, hy0, ldhy0);
}

}  // namespace chfsi

extern "C" {

int chfsi_debug_k1_trace(unsigned long long* host, int max_ctas) {
  CK_ARG(host && max_ctas >= 0, "bad argument");
  const int n = chfsi::step_trace_copy(host, max_ctas);
  if (n < 0) return fail(CHFSI_ECUDA, "trace copy failed");
  return n;
}

int chfsi_step_tiling(int n, int w, int* bm, int* bn, int* split) {
  CK_ARG(bm && bn && split, "NULL output");
  const chfsi::StepTiling t = chfsi::choose_step_tiling(n, w);
  *bm = t.bm;
  *bn = t.bn;
  *split = t.split;
  return CHFSI_OK;
}

int chfsi_set_complex_product(int product) {
  if (product == 0) return chfsi::complex_product();
  CK_ARG(product == 3 || product == 4, "complex product must be 3 or 4");
  return chfsi::set_complex_product(product);
}

int chfsi_set_panel_kernels(int on) {
  CK_ARG(on == -1 || on == 0 || on == 1, "panel kernels: 1 on, 0 off, -1 query");
  if (on == -1) return chfsi::g_panel_kernels.load(std::memory_order_relaxed) ? 1 : 0;
  return chfsi::g_panel_kernels.exchange(on != 0) ? 1 : 0;
}

int chfsi_set_k1_slab(int halves) {
  CK_ARG(halves == 0 || halves == 2 || halves == 4, "k-slab depth must be 2 or 4 halves");
  if (halves == 0) {  // query
    const int cur = chfsi::set_k1_slab(2);
    chfsi::set_k1_slab(cur);
    return cur;
  }
  return chfsi::set_k1_slab(halves);
}

// ------------------------------------------------------------------- K2 ---

int chfsi_lanczos_z(chfsi_ctx* ctx, int n, int k, const void* H, long long ldh, int conj_h,
                    const void* q0, void* basis, double* alphas, double* betas, double* beta_last,
                    int* steps) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(n >= 1 && k >= 1 && k <= n, "need 1 <= k <= n");
  CK_ARG(H && q0 && basis && alphas && betas && beta_last && steps, "NULL argument");
  if (ctx->lanczos_mode == 0) {  // one cooperative persistent kernel (lanczos.cu)
    const size_t ws = chfsi::lanczos_coop_workspace_bytes(n, k);
    CK(ensure_scratch(ctx, ws + 2 * (size_t)k * sizeof(double) + 256));
    double* al_d = reinterpret_cast<double*>(static_cast<char*>(ctx->scratch) + ws);
    double* be_d = al_d + k;
    cudaStream_t s = ctx->stream;
    CK_CUDA(cudaMemsetAsync(ctx->lstate, 0, sizeof(LanczosState), s));
    CK_CUDA(cudaMemsetAsync(be_d, 0, (size_t)k * sizeof(double), s));
    CK_CUDA(chfsi::lanczos_coop_launch(static_cast<const double2*>(H), ldh, conj_h != 0, n, k,
                                       static_cast<const double2*>(q0), static_cast<double2*>(basis),
                                       ctx->scratch, al_d, be_d, ctx->lstate, s));
    LanczosState hst;
    CK_CUDA(cudaMemcpyAsync(&hst, ctx->lstate, sizeof(hst), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaMemcpyAsync(alphas, al_d, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaMemcpyAsync(betas, be_d, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaStreamSynchronize(s));
    *steps = hst.steps;
    *beta_last = hst.beta_last;
    return CHFSI_OK;
  }
  // multi-kernel path (reference for tests): u, r (n each), coef (k), alphas_d, betas_d (k)
  const size_t vec = (size_t)n * sizeof(double2);
  CK(ensure_scratch(ctx, 2 * vec + (size_t)k * sizeof(double2) + 2 * (size_t)k * sizeof(double) + 256));
  char* base = static_cast<char*>(ctx->scratch);
  double2* u = reinterpret_cast<double2*>(base);
  double2* r = reinterpret_cast<double2*>(base + vec);
  double2* coef = reinterpret_cast<double2*>(base + 2 * vec);
  double* al_d = reinterpret_cast<double*>(base + 2 * vec + (size_t)k * sizeof(double2));
  double* be_d = al_d + k;
  double2* V = static_cast<double2*>(basis);
  const double2* hh = static_cast<const double2*>(H);
  cudaStream_t s = ctx->stream;
  LanczosState* st = ctx->lstate;
  const int* done = &st->done;
  double* nrm = ctx->scalars;
  CK_CUDA(cudaMemsetAsync(st, 0, sizeof(LanczosState), s));
  CK_CUDA(cudaMemsetAsync(be_d, 0, (size_t)k * sizeof(double), s));
  // q = q0 / ||q0||  (chfsi.py:137-138)
  CK_CUDA(chfsi::norm2_launch(static_cast<const double2*>(q0), n, ctx->partial, nrm, nullptr, s));
  CK_CUDA(chfsi::div_scalar_launch(static_cast<const double2*>(q0), nrm, V, n, s));
  for (int i = 0; i < k; ++i) {
    const double2* q = V + (long long)i * n;
    CK_CUDA(chfsi::gemv_rows_launch(hh, ldh, conj_h != 0, q, u, n, done, s));
    CK_CUDA(chfsi::dot_re_launch(q, u, n, ctx->partial, al_d + i, done, s));
    CK_CUDA(chfsi::lanczos_residual_launch(u, q, i ? V + (long long)(i - 1) * n : nullptr,
                                           al_d + i, i ? be_d + i - 1 : nullptr, r, n, done, s));
    CK_CUDA(chfsi::colsdot_launch(V, n, n, i + 1, r, coef, done, s));
    CK_CUDA(chfsi::sub_vcoef_launch(V, n, n, i + 1, coef, r, done, s));
    CK_CUDA(chfsi::norm2_launch(r, n, ctx->partial, nrm, done, s));
    CK_CUDA(chfsi::lanczos_advance_launch(r, nrm, i + 1 < k ? V + (long long)(i + 1) * n : nullptr,
                                          be_d + i, st, i, k, n, s));
  }
  LanczosState hst;
  CK_CUDA(cudaMemcpyAsync(&hst, st, sizeof(hst), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaMemcpyAsync(alphas, al_d, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaMemcpyAsync(betas, be_d, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaStreamSynchronize(s));
  *steps = hst.steps;
  *beta_last = hst.beta_last;
  return CHFSI_OK;
}

// ------------------------------------------------------------ K3 / K4 ---

int chfsi_gemm_z(chfsi_ctx* ctx, char transa, char transb, int m, int n, int k, double alpha_re,
                 double alpha_im, const void* A, long long lda, const void* B, long long ldb,
                 double beta_re, double beta_im, void* C, long long ldc) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(valid_op(transa) && valid_op(transb), "unknown transpose flag");
  CK_ARG(m >= 0 && n >= 0 && k >= 0, "negative size");
  if (m == 0 || n == 0) return CHFSI_OK;
  // (Measured and rejected, round 2: Gram-type products C = A^H B of the loop
  // — CGS coefficients, Cholesky-QR Grams, the projected matrix — on K1's
  // stream-K schedule, A's columns read conjugated through TMA. Correct and
  // deterministic, but the ~20-way fixed-order fold per output tile costs
  // more than cuBLAS's z884gemm + splitKreduce pair: C2 ortho 31 -> 39 ms.)
  const cuDoubleComplex al = make_cuDoubleComplex(alpha_re, alpha_im);
  const cuDoubleComplex be = make_cuDoubleComplex(beta_re, beta_im);
  CK_BLAS(cublasZgemm(ctx->blas, op_of(transa), op_of(transb), m, n, k, &al,
                      static_cast<const cuDoubleComplex*>(A), (int)lda,
                      static_cast<const cuDoubleComplex*>(B), (int)ldb, &be,
                      static_cast<cuDoubleComplex*>(C), (int)ldc));
  return CHFSI_OK;
}

int chfsi_cgs_project_z(chfsi_ctx* ctx, int n, int nlocked, int w, const void* locked,
                        long long ldl, void* work, long long ldw, void* coef) {
  CK_ARG(ctx, "ctx is NULL");
  if (nlocked == 0 || w == 0 || n == 0) return CHFSI_OK;
  for (int pass = 0; pass < 2; ++pass) {
    CK(chfsi_gemm_z(ctx, 'C', 'N', nlocked, w, n, 1.0, 0.0, locked, ldl, work, ldw, 0.0, 0.0,
                    coef, nlocked));
    CK(chfsi_gemm_z(ctx, 'N', 'N', n, w, nlocked, -1.0, 0.0, locked, ldl, coef, nlocked, 1.0,
                    0.0, work, ldw));
  }
  return CHFSI_OK;
}

}  // extern "C"

namespace {

// Householder QR (cuSOLVER geqrf/ungqr) with the reference's rank test and
// positive-real R diagonal (linalg.py:152-178). y holds Y on entry, Q on
// success; on rank deficiency y is restored from `backup`.
int qr_householder(chfsi_ctx* ctx, int m, int n, double2* y, const double2* backup, double2* tau,
                   double2* rdiag, const double* fro, int* dead, int* ndead) {
  cudaStream_t s = ctx->stream;
  const size_t blk = (size_t)m * n * sizeof(double2);
  int lwork = 0, lwork2 = 0;
  CK_SOLVER(cusolverDnZgeqrf_bufferSize(ctx->solver, m, n, reinterpret_cast<cuDoubleComplex*>(y),
                                        m, &lwork));
  CK_SOLVER(cusolverDnZungqr_bufferSize(ctx->solver, m, n, n,
                                        reinterpret_cast<cuDoubleComplex*>(y), m,
                                        reinterpret_cast<cuDoubleComplex*>(tau), &lwork2));
  if (lwork2 > lwork) lwork = lwork2;
  CK(ensure_ws(ctx, (size_t)lwork * sizeof(cuDoubleComplex)));
  CK_SOLVER(cusolverDnZgeqrf(ctx->solver, m, n, reinterpret_cast<cuDoubleComplex*>(y), m,
                             reinterpret_cast<cuDoubleComplex*>(tau),
                             static_cast<cuDoubleComplex*>(ctx->ws), lwork, ctx->dinfo));
  CK_CUDA(chfsi::extract_diag_launch(y, m, n, rdiag, s));
  std::vector<double2> hd(n);
  double hfro = 0.0;
  CK_CUDA(cudaMemcpyAsync(hd.data(), rdiag, (size_t)n * sizeof(double2), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaMemcpyAsync(&hfro, fro, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaStreamSynchronize(s));
  const double thresh = 1e-13 * hfro;  // linalg.py:173
  int nd = 0;
  for (int j = 0; j < n; ++j)
    if (std::hypot(hd[j].x, hd[j].y) < thresh) dead[nd++] = j;
  if (nd) {
    *ndead = nd;
    CK_CUDA(cudaMemcpyAsync(y, backup, blk, cudaMemcpyDeviceToDevice, s));
    return fail(CHFSI_ERANK, "rank-deficient columns");
  }
  CK_SOLVER(cusolverDnZungqr(ctx->solver, m, n, n, reinterpret_cast<cuDoubleComplex*>(y), m,
                             reinterpret_cast<cuDoubleComplex*>(tau),
                             static_cast<cuDoubleComplex*>(ctx->ws), lwork, ctx->dinfo));
  CK_CUDA(chfsi::phase_fix_launch(y, m, m, n, rdiag, s));
  return CHFSI_OK;
}

// linear2: the second of two passes is linearised — after a first pass Q1 is
// orthonormal to eps = max|Q1^H Q1 - I| ~ u cond(Y)^2 (~1e-13 for the filtered
// panels), and for G = I + E the Cholesky factor is R2 = I + tri(E) + O(eps^2)
// (tri = strict upper + diag/2), so Q = Q1 (I - tri(E)) has Q^H Q = I +
// O(eps^2): one ZGEMM Gram, one small kernel and one ZGEMM replace
// potrf + ZTRSM (2048 x 160: ~145 -> ~35 us). Accepted only when eps <= 1e-8
// (*linear_reject otherwise; the caller reruns the exact pass).
int qr_cholqr(chfsi_ctx* ctx, int m, int n, double2* y, double2* g, double* rdiag_acc,
              double* rlast, const double* fro, int passes, bool shifted, bool* fallback,
              double* last_dev, bool linear2 = false, bool* linear_reject = nullptr,
              double2* tmp = nullptr, bool defer = false) {
  cudaStream_t s = ctx->stream;
  *fallback = false;
  *last_dev = 0.0;
  if (linear_reject) *linear_reject = false;
  linear2 = linear2 && passes == 2 && !shifted && tmp != nullptr;
  // The acceptance test's inputs are contiguous on the device in the order
  // the host reads them — [rdiag_acc n | fro | rlast n | eps | info] (the
  // callers lay the scratch out so) — and come back in ONE copy per call.
  CK_ARG(rlast == rdiag_acc + n + 1 && fro == rdiag_acc + n, "qr_cholqr scratch layout");
  double* eps_dev = rlast + n;
  int* info_dev = reinterpret_cast<int*>(rlast + n + 1);
  // The factor is taken LOWER (G = L L^H, L = R^H) and Y <- Y L^-H: cuSOLVER's
  // lower potrf is ~1.8x faster than its upper one at the panel sizes (w=160:
  // 74 vs 135 us, tools/microbench/qr_bench.cu); the TRSM costs the same.
  int lwork = 0;
  CK_SOLVER(cusolverDnZpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, n,
                                        reinterpret_cast<cuDoubleComplex*>(g), n, &lwork));
  CK(ensure_ws(ctx, (size_t)lwork * sizeof(cuDoubleComplex)));
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  // unit roundoff 2^-53; Fukaya's shift 11 (mn + n(n+1)) u ||Y||_2^2 with ||Y||_F >= ||Y||_2
  const double shift_coef = 11.0 * ((double)m * n + (double)n * (n + 1)) * 1.1102230246251565e-16;
  // Shape-dependent library choices (profiles/r01_qr_bench.log): the Gram by
  // ZHERK from w >= 1000 (12000 x 1400: 3.2 vs 5.3 ms; ZGEMM wins below, e.g.
  // 2048 x 160: 25 vs 76 us), and the linearised pass's Q1 M by out-of-place
  // ZTRMM from w >= 400 (5000 x 600: 0.28 vs 0.43 ms; 2048 x 160: ZGEMM 23 vs 26 us).
  const bool herk = n >= 1000, trmm = n >= 400;
  // Panel widths of the ChFSI loop (n <= kPanelMaxW): the triangular solve
  // and the linearised pass run as one row-parallel kernel each
  // (panel_kernels.cu) instead of cuBLAS's latency-bound ZTRSM chain and
  // near-identity update + ZGEMM + copy-back (2048 x 160 in the C2 loop:
  // ~47 + ~45 us -> ~2 x 10 us). CHFSI_PANEL_KERNELS=0 restores the
  // library calls.
  const bool panel = chfsi::g_panel_kernels.load(std::memory_order_relaxed) && n <= chfsi::kPanelMaxW;
  if (panel && !ctx->panel_linv) CK_CUDA(cudaMalloc(&ctx->panel_linv, chfsi::panel_linv_bytes()));
  for (int pass = 0; pass < passes; ++pass) {
    const bool lin = linear2 && pass == 1;
    if (herk) {  // lower triangle for potrf, upper for the near-identity kernel
      const double done = 1.0, dzero = 0.0;
      CK_BLAS(cublasZherk(ctx->blas, lin ? CUBLAS_FILL_MODE_UPPER : CUBLAS_FILL_MODE_LOWER,
                          CUBLAS_OP_C, n, m, &done, reinterpret_cast<const cuDoubleComplex*>(y), m,
                          &dzero, reinterpret_cast<cuDoubleComplex*>(g), n));
    } else {
      CK(chfsi_gemm_z(ctx, 'C', 'N', n, n, m, 1.0, 0.0, y, m, y, m, 0.0, 0.0, g, n));
    }
    if (shifted && pass == 0) CK_CUDA(chfsi::add_diag_shift_launch(g, n, n, fro, shift_coef, s));
    if (linear2 && pass == 1 && panel) {
      CK_CUDA(chfsi::panel_apply_near_identity_launch(y, m, m, n, g, n, rdiag_acc, rlast, eps_dev, s));
      continue;
    }
    if (linear2 && pass == 1) {
      CK_CUDA(chfsi::near_identity_update_launch(g, n, n, rdiag_acc, rlast, eps_dev, s));
      // Q = Q1 M out of place (ZGEMM + copy back: 2048 x 160 27 us vs 47 us
      // for cuBLAS's in-place ZTRMM; M's strict lower triangle is zero)
      if (trmm)
        CK_BLAS(cublasZtrmm(ctx->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                            CUBLAS_DIAG_NON_UNIT, m, n, &one, reinterpret_cast<const cuDoubleComplex*>(g),
                            n, reinterpret_cast<const cuDoubleComplex*>(y), m,
                            reinterpret_cast<cuDoubleComplex*>(tmp), m));
      else
        CK_BLAS(cublasZgemm(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_N, m, n, n, &one,
                            reinterpret_cast<const cuDoubleComplex*>(y), m,
                            reinterpret_cast<const cuDoubleComplex*>(g), n, &zero,
                            reinterpret_cast<cuDoubleComplex*>(tmp), m));
      CK_CUDA(cudaMemcpyAsync(y, tmp, (size_t)m * n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      continue;
    }
    CK_SOLVER(cusolverDnZpotrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, n,
                               reinterpret_cast<cuDoubleComplex*>(g), n,
                               static_cast<cuDoubleComplex*>(ctx->ws), lwork, info_dev + pass));
    if (panel) {
      CK_CUDA(chfsi::panel_post_potrf_launch(g, n, n, rdiag_acc, pass == 0,
                                             pass == passes - 1 ? rlast : nullptr, ctx->panel_linv,
                                             linear2 ? eps_dev : nullptr, s));
      CK_CUDA(chfsi::panel_trsm_lh_launch(y, m, m, n, g, n, ctx->panel_linv, s));
      continue;
    }
    CK_CUDA(chfsi::diag_accumulate_launch(g, n, n, rdiag_acc, pass == 0, s));
    if (pass == passes - 1) CK_CUDA(chfsi::diag_accumulate_launch(g, n, n, rlast, true, s));
    CK_BLAS(cublasZtrsm(ctx->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C,
                        CUBLAS_DIAG_NON_UNIT, m, n, &one, reinterpret_cast<const cuDoubleComplex*>(g),
                        n, reinterpret_cast<cuDoubleComplex*>(y), m));
  }
  const size_t hbytes = (size_t)(2 * n + 2) * sizeof(double) + 4 * sizeof(int);
  if (defer && hbytes > ctx->qr_pinned_bytes) {
    CK_CUDA(cudaStreamSynchronize(s));
    if (ctx->qr_pinned) CK_CUDA(cudaFreeHost(ctx->qr_pinned));
    ctx->qr_pinned = nullptr;
    ctx->qr_pinned_bytes = 0;
    CK_CUDA(cudaMallocHost(&ctx->qr_pinned, std::max<size_t>(hbytes, 4096)));
    ctx->qr_pinned_bytes = std::max<size_t>(hbytes, 4096);
  }
  if (!defer) CK(chfsi::ensure_pinned(ctx, hbytes));
  double* hd = static_cast<double*>(defer ? ctx->qr_pinned : ctx->pinned);
  double* hl = hd + n + 1;
  double* heps = hl + n;
  int* info = reinterpret_cast<int*>(heps + 1);
  CK_CUDA(cudaMemcpyAsync(hd, rdiag_acc, hbytes, cudaMemcpyDeviceToHost, s));
  if (defer) {  // judged later by qr_deferred_verdict (same checks as below)
    ctx->qr_pending = true;
    ctx->qr_pending_n = n;
    *fallback = false;
    *last_dev = 0.0;
    return CHFSI_OK;
  }
  CK_CUDA(cudaStreamSynchronize(s));
  const double hfro = hd[n];
  bool bad = !std::isfinite(hfro);
  for (int pass = 0; pass < (linear2 ? 1 : passes); ++pass) bad = bad || info[pass] != 0;
  if (bad) {
    *fallback = true;
    return CHFSI_OK;
  }
  const double safe = 1e-11 * hfro;
  double dev = 0.0;
  for (int j = 0; j < n; ++j) {
    if (!(hd[j] >= safe)) {  // also catches NaN
      *fallback = true;
      return CHFSI_OK;
    }
    dev = std::max(dev, std::fabs(hl[j] - 1.0));
  }
  *last_dev = std::isfinite(dev) ? dev : INFINITY;
  if (linear2 && !(*heps <= 1e-8)) {  // also NaN: rerun the pass exactly
    *fallback = true;
    if (linear_reject) *linear_reject = true;
  }
  return CHFSI_OK;
}

}  // namespace

extern "C" {

int chfsi_qr_orthonormalize_z(chfsi_ctx* ctx, int m, int n, void* Y, long long ldy, int* dead,
                              int* ndead) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(m >= n && n >= 0, "need rows >= cols");
  CK_ARG(ndead && dead, "NULL output");
  *ndead = 0;
  if (n == 0) return CHFSI_OK;
  CK_ARG(ldy == m, "QR needs a packed block (ldy == m)");
  cudaStream_t s = ctx->stream;
  double2* y = static_cast<double2*>(Y);
  // scratch: backup copy of Y (m*n), tau (n), rdiag (n), Gram (n*n), diag accumulator (n),
  // last pass's diagonal (n)
  const size_t blk = (size_t)m * n * sizeof(double2);
  CK(ensure_scratch(ctx, 2 * blk + 2 * (size_t)n * sizeof(double2) + (size_t)n * n * sizeof(double2) +
                             (2 * (size_t)n + 4) * sizeof(double)));
  double2* backup = static_cast<double2*>(ctx->scratch);
  double2* tau = backup + (size_t)m * n;
  double2* rdiag = tau + n;
  double2* g = rdiag + n;
  // [racc n | fro | rlast n | eps | info]: the acceptance test's inputs (qr_cholqr)
  double* racc = reinterpret_cast<double*>(g + (size_t)n * n);
  double* fro = racc + n;
  double* rlast = racc + n + 1;
  double2* tmp = reinterpret_cast<double2*>(racc + 2 * (size_t)n + 4);  // m x n (linearised pass 2)
  CK_CUDA(chfsi::copy_norm2_launch(y, backup, (long long)m * n, ctx->partial, ctx->red_counter, fro, s));
  if (ctx->qr_mode != 1) {  // 0: Cholesky-QR first, 1: Householder only
    bool fallback = false;
    double dev = 0.0;
    // Cholesky-QR2 (no shift) accepts when the second pass's R is the
    // identity to 1e-6, i.e. the first pass already left Q within 1e-6 of
    // orthonormal: the second pass then makes it orthonormal to rounding.
    // The filtered panels are well conditioned (R diagonal ranges <= 50 over
    // the C2 sequence), so this is the common case; otherwise the shifted
    // Cholesky-QR3 runs from the backup, and Householder after that.
    if (ctx->qr_mode == 0) {
      bool lin_reject = false;
      CK(qr_cholqr(ctx, m, n, y, g, racc, rlast, fro, 2, false, &fallback, &dev,
                   ctx->qr_linear2, &lin_reject, tmp));
      if (!fallback && dev <= 1e-6) return CHFSI_OK;
      CK_CUDA(cudaMemcpyAsync(y, backup, blk, cudaMemcpyDeviceToDevice, s));
      if (lin_reject) {  // the first pass was fine but left |Q1^H Q1 - I| > 1e-8: exact pass 2
        CK(qr_cholqr(ctx, m, n, y, g, racc, rlast, fro, 2, false, &fallback, &dev));
        if (!fallback && dev <= 1e-6) return CHFSI_OK;
        CK_CUDA(cudaMemcpyAsync(y, backup, blk, cudaMemcpyDeviceToDevice, s));
      }
    }
    CK(qr_cholqr(ctx, m, n, y, g, racc, rlast, fro, 3, true, &fallback, &dev));
    if (!fallback) return CHFSI_OK;
    CK_CUDA(cudaMemcpyAsync(y, backup, blk, cudaMemcpyDeviceToDevice, s));
  }
  return qr_householder(ctx, m, n, y, backup, tau, rdiag, fro, dead, ndead);
}

}  // extern "C"

namespace chfsi {

int qr_orthonormalize_deferred(chfsi_ctx* ctx, int m, int n, void* Y, long long ldy) {
  CK_ARG(ctx && Y && m >= n && n >= 1 && ldy == m, "bad deferred QR arguments");
  CK_ARG(ctx->qr_mode == 0 && ctx->qr_linear2, "the deferred QR is the default Cholesky-QR2 only");
  cudaStream_t s = ctx->stream;
  double2* y = static_cast<double2*>(Y);
  const size_t blk = (size_t)m * n * sizeof(double2);
  CK(ensure_scratch(ctx, 2 * blk + 2 * (size_t)n * sizeof(double2) + (size_t)n * n * sizeof(double2) +
                             (2 * (size_t)n + 4) * sizeof(double)));
  double2* backup = static_cast<double2*>(ctx->scratch);
  double2* g = backup + (size_t)m * n + 2 * (size_t)n;
  double* racc = reinterpret_cast<double*>(g + (size_t)n * n);  // [racc n | fro | rlast n | eps | info]
  double* fro = racc + n;
  double* rlast = racc + n + 1;
  double2* tmp = reinterpret_cast<double2*>(racc + 2 * (size_t)n + 4);
  CK_CUDA(chfsi::copy_norm2_launch(y, backup, (long long)m * n, ctx->partial, ctx->red_counter, fro, s));
  bool fallback = false, lin_reject = false;
  double dev = 0.0;
  return qr_cholqr(ctx, m, n, y, g, racc, rlast, fro, 2, false, &fallback, &dev, true,
                   &lin_reject, tmp, /*defer=*/true);
}

int qr_deferred_verdict(chfsi_ctx* ctx, bool* accept) {
  CK_ARG(ctx && accept && ctx->qr_pending, "no deferred QR pending");
  ctx->qr_pending = false;
  const int n = ctx->qr_pending_n;
  const double* hd = static_cast<const double*>(ctx->qr_pinned);
  const double* hl = hd + n + 1;
  const double heps = hl[n];
  const int* info = reinterpret_cast<const int*>(hl + n + 1);
  const double hfro = hd[n];
  // the checks of qr_cholqr + chfsi_qr_orthonormalize_z's acceptance (linearised CholQR2)
  bool ok = std::isfinite(hfro) && info[0] == 0;
  const double safe = 1e-11 * hfro;
  double dev = 0.0;
  for (int j = 0; ok && j < n; ++j) {
    if (!(hd[j] >= safe)) ok = false;  // also NaN
    dev = std::max(dev, std::fabs(hl[j] - 1.0));
  }
  ok = ok && std::isfinite(dev) && dev <= 1e-6 && heps <= 1e-8;
  *accept = ok;
  return CHFSI_OK;
}

int qr_deferred_restore(chfsi_ctx* ctx, int m, int n, void* Y) {
  CK_CUDA(cudaMemcpyAsync(Y, ctx->scratch, (size_t)m * n * sizeof(double2), cudaMemcpyDeviceToDevice,
                          ctx->stream));
  return CHFSI_OK;
}

}  // namespace chfsi

extern "C" {

int chfsi_ctx_set_lanczos_mode(chfsi_ctx* ctx, int mode) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(mode == 0 || mode == 1, "lanczos mode must be 0 (cooperative) or 1 (multi-kernel)");
  ctx->lanczos_mode = mode;
  return CHFSI_OK;
}

int chfsi_ctx_set_qr_linear2(chfsi_ctx* ctx, int on) {
  CK_ARG(ctx, "ctx is NULL");
  ctx->qr_linear2 = on != 0;
  return CHFSI_OK;
}

int chfsi_ctx_set_qr_mode(chfsi_ctx* ctx, int mode) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(mode >= 0 && mode <= 2,
         "qr mode must be 0 (Cholesky-QR2, then shifted Cholesky-QR3, then Householder), "
         "1 (Householder) or 2 (shifted Cholesky-QR3, then Householder)");
  ctx->qr_mode = mode;
  return CHFSI_OK;
}

}  // extern "C"

namespace {

// Near-diagonal Hermitian eigensolver (nd_eig.cu): simultaneous first-order
// Jacobi steps X = I + S, S_ij = G_ij / (d_j - d_i); W <- W X made unitary by
// Newton-Schulz polar iterations; G = W^H G0 W projected exactly from the
// input, so G stays unitarily similar to it and the off-diagonal/gap ratio r
// squares every step. Adaptive: after each step's O(w^2) measurement the host
// stops as soon as max|G_ij| <= tol * max(1, max|G_ii|), and the number of
// NS iterations follows r (the unitarity defect of W X is ~|S|^2 and squares
// per NS iteration). *done = false (A untouched) when G is not in that regime
// (r > 0.5, CHFSI_RR_BAIL), does not converge within kMaxSteps, or W is not unitary to
// rounding (defect at the last NS input > 1e-8): the caller uses zheevd.
double nd_bail() {  // regime bound on max|G_ij| / |d_j - d_i| (tuning)
  static const double bail = [] {
    const char* e = getenv("CHFSI_RR_BAIL");
    return e ? atof(e) : 0.5;  // measured: 0.1 -> 0.5 turns 5 of the cold C2 start's 10 zheevd calls into fast ones
  }();
  return bail;
}

bool nd_persist_enabled() {
  static const bool persist = [] {
    const char* e = getenv("CHFSI_ND_PERSIST");
    return !(e && atoi(e) == 0);
  }();
  return persist;
}

// The cooperative near-diagonal eigensolver (nd_persist.cu) queued on the
// stream with its 4-double status copied to page-locked `hs` — no host
// synchronisation here.
int nd_persist_queue(chfsi_ctx* ctx, int n, double2* a, long long lda, double* w, double tol, double* hs) {
  cudaStream_t s = ctx->stream;
  const size_t pneed = chfsi::nd_persist_ws_bytes(n);
  if (pneed > ctx->eig_ws_bytes) {
    CK_CUDA(cudaStreamSynchronize(s));
    if (ctx->eig_ws) CK_CUDA(cudaFree(ctx->eig_ws));
    ctx->eig_ws = nullptr;
    ctx->eig_ws_bytes = 0;
    CK_CUDA(cudaMalloc(&ctx->eig_ws, pneed));
    ctx->eig_ws_bytes = pneed;
  }
  double* st_dev = ctx->scalars + 12;  // 4 doubles of the context's scalar scratch
  CK_CUDA(chfsi::nd_persist_launch(a, lda, n, w, tol, nd_bail(), ctx->eig_ws, st_dev, s));
  CK_CUDA(cudaMemcpyAsync(hs, st_dev, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
  return CHFSI_OK;
}

int heev_near_diag(chfsi_ctx* ctx, int n, double2* a, long long lda, double* w, double tol,
                   bool* done) {
  *done = false;
  cudaStream_t s = ctx->stream;
  const size_t mat = (size_t)n * n * sizeof(double2);
  constexpr int kMaxSteps = 6;
  const double bail = nd_bail();
  constexpr int kSlots = 4 * (kMaxSteps + 1) + kMaxSteps;  // build stats + NS defects
  // Panel widths: the whole iteration as one cooperative kernel (nd_persist.cu;
  // CHFSI_ND_PERSIST=0 keeps the multi-kernel version below) — one host
  // round trip per call instead of one per step, no per-step launches.
  if (nd_persist_enabled() && n <= chfsi::kNdPersistMaxN) {
    CK(chfsi::ensure_pinned(ctx, 4 * sizeof(double)));
    double* hs = static_cast<double*>(ctx->pinned);
    CK(nd_persist_queue(ctx, n, a, lda, w, tol, hs));
    CK_CUDA(cudaStreamSynchronize(s));
    static const bool dbgp = getenv("CHFSI_RR_DEBUG") != nullptr;
    if (dbgp)
      fprintf(stderr, "ndp n=%d done=%g steps=%g rmax=%.3e emax=%.3e\n", n, hs[0], hs[1], hs[2], hs[3]);
    *done = hs[0] == 1.0;
    return CHFSI_OK;
  }
  const size_t need = 5 * mat + kSlots * sizeof(double) + (size_t)n * sizeof(int) + 1024;
  if (need > ctx->eig_ws_bytes) {
    CK_CUDA(cudaStreamSynchronize(s));
    if (ctx->eig_ws) CK_CUDA(cudaFree(ctx->eig_ws));
    ctx->eig_ws = nullptr;
    ctx->eig_ws_bytes = 0;
    CK_CUDA(cudaMalloc(&ctx->eig_ws, need));
    ctx->eig_ws_bytes = need;
  }
  CK(chfsi::ensure_pinned(ctx, kSlots * sizeof(double)));
  double2* G0 = reinterpret_cast<double2*>(ctx->eig_ws);  // the input, kept for the exact projection
  double2* G = G0 + (size_t)n * n;                          // working iterate
  double2* X = G + (size_t)n * n;
  double2* Y = X + (size_t)n * n;
  double2* W = Y + (size_t)n * n;                           // accumulated eigenvector basis
  double* stats = reinterpret_cast<double*>(W + (size_t)n * n);  // [step][4], then [step] NS defect
  double* defect = stats + 4 * (kMaxSteps + 1);
  int* perm = reinterpret_cast<int*>(stats + kSlots);
  double* hs = static_cast<double*>(ctx->pinned);
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  auto gemm = [&](cublasOperation_t ta, const double2* A_, const double2* B_, double2* C_) -> int {
    CK_BLAS(cublasZgemm(ctx->blas, ta, CUBLAS_OP_N, n, n, n, &one,
                        reinterpret_cast<const cuDoubleComplex*>(A_), n,
                        reinterpret_cast<const cuDoubleComplex*>(B_), n, &zero,
                        reinterpret_cast<cuDoubleComplex*>(C_), n));
    return CHFSI_OK;
  };
  CK_CUDA(cudaMemsetAsync(stats, 0, kSlots * sizeof(double), s));
  CK_CUDA(chfsi::copy_cols_launch(a, lda, G0, n, n, n, s));
  const double2* Gcur = G0;  // step 0 measures the input directly
  double last_defect = 0.0;
  for (int it = 0;; ++it) {
    CK_CUDA(chfsi::nd_build_step_launch(Gcur, n, n, X, n, stats + 4 * it, s));
    CK_CUDA(cudaMemcpyAsync(hs, stats + 4 * it, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (it > 0)
      CK_CUDA(cudaMemcpyAsync(hs + 4, defect + it - 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaStreamSynchronize(s));
    const double rmax = hs[0], emax = hs[1], dmax = hs[2];
    static const bool dbg = getenv("CHFSI_RR_DEBUG") != nullptr;  // diagnostics: regime per step
    if (dbg) fprintf(stderr, "nd n=%d it=%d rmax=%.3e emax=%.3e dmax=%.3e\n", n, it, rmax, emax, dmax);
    if (it > 0) last_defect = hs[4];
    if (it > 0 && emax <= tol * std::max(1.0, dmax)) {
      if (!(last_defect <= 1e-8)) return CHFSI_OK;  // W not unitary to rounding: zheevd
      break;
    }
    if (it == kMaxSteps || !(rmax <= bail)) return CHFSI_OK;  // not near-diagonal / not converging
    if (it == 0) {
      std::swap(W, X);  // W = X
    } else {
      CK(gemm(CUBLAS_OP_N, W, X, Y));
      std::swap(W, Y);  // W = W X
    }
    // unitarity defect of W X ~ |S|^2 <~ (sqrt(n) r)^2, squared by each NS step
    const double sr = std::sqrt((double)n) * rmax;
    const int ns = sr <= 5e-5 ? 1 : (sr <= 7e-3 ? 2 : (sr <= 0.08 ? 3 : (sr <= 0.3 ? 4 : 5)));
    for (int k = 0; k < ns; ++k) {  // W <- W (3I - W^H W) / 2
      CK(gemm(CUBLAS_OP_C, W, W, Y));
      CK_CUDA(chfsi::nd_ns_matrix_launch(Y, n, n, k == ns - 1 ? defect + it : nullptr, s));
      CK(gemm(CUBLAS_OP_N, W, Y, X));
      std::swap(W, X);
    }
    CK(gemm(CUBLAS_OP_N, G0, W, X));  // X = G0 W
    CK(gemm(CUBLAS_OP_C, W, X, G));   // G = W^H G0 W
    CK_CUDA(chfsi::symmetrize_launch(G, n, n, s));
    Gcur = G;
  }
  // ascending eigenvalues, eigenvectors permuted accordingly, back into A
  CK_CUDA(chfsi::nd_sort_launch(G, n, n, w, perm, s));
  CK_CUDA(chfsi::nd_gather_cols_launch(W, n, n, n, perm, a, lda, s));
  *done = true;
  return CHFSI_OK;
}

}  // namespace

namespace chfsi {

int heev_rr_speculative(chfsi_ctx* ctx, int n, void* A, long long lda, double* w, double tol, bool* queued) {
  *queued = false;
  if (!(tol > 0.0) || n < 2 || n > kNdPersistMaxN || !nd_persist_enabled()) return CHFSI_OK;
  if (!ctx->nd_pinned) CK_CUDA(cudaMallocHost(&ctx->nd_pinned, 4 * sizeof(double)));
  CK(nd_persist_queue(ctx, n, static_cast<double2*>(A), lda, w, tol, ctx->nd_pinned));
  ctx->nd_pending = true;
  *queued = true;
  return CHFSI_OK;
}

int heev_rr_verdict(chfsi_ctx* ctx, bool* done) {
  CK_ARG(ctx && done && ctx->nd_pending, "no speculative eigensolver pending");
  ctx->nd_pending = false;
  *done = ctx->nd_pinned[0] == 1.0;
  return CHFSI_OK;
}

}  // namespace chfsi

namespace {

// Block size of the K1-based triangular solves (tuning: CHFSI_TRSM_NB).
int trsm_nb() {
  static const int nb = [] {
    const char* e = getenv("CHFSI_TRSM_NB");
    const int v = e ? atoi(e) : 256;
    return v >= 32 ? v : 256;
  }();
  return nb;
}

// One K1 update on rows [r0, r0 + rows) of the n x m block R:
//   R[r0:r0+rows, :] -= op(A) R[k0:k0+kc, :],  op(A)[r][k] = conj(S[(r0+r)*lds + k])
// (S's column r0 + r, rows k0.., conjugated: the rows of L read through L^H's
// column-major storage, or the rows of L^H through L's) — the epilogue
// Ynext = alpha (acc - 0) - beta Yprev with alpha = beta = -1, in place.
int k1_block_update(chfsi_ctx* ctx, int n, int m, const double2* S, long long lds, int r0, int rows,
                    int k0, int kc, double2* R, long long ldr) {
  if (kc <= 0 || rows <= 0 || m <= 0) return CHFSI_OK;
  const chfsi::RowShard shard{rows, 0, 0, nullptr, 0};
  chfsi::StepTiling tiling = chfsi::choose_step_tiling(n, m);
  // few output tiles over a long contraction (the back-transform's 256 x nev
  // blocks): cap the stream-K split at 4 CTAs per tile — spread over every
  // resident CTA each owner folds dozens of partial tiles (37 -> ~15 us)
  const long long tiles = (long long)((rows + tiling.bm - 1) / tiling.bm) * ((m + tiling.bn - 1) / tiling.bn);
  if (tiles * 4 < chfsi::kNumSMs) tiling.split = (int)(tiles * 4);
  CK_CUDA(chfsi::cheb_step_rows_launch(S + (long long)r0 * lds + k0, lds, /*conj=*/true, R + k0, ldr,
                                       R + r0, ldr, R + r0, ldr, kc, m, -1.0, 0.0, -1.0, shard, tiling,
                                       ctx->step_ws, ctx->stream));
  return CHFSI_OK;
}

// L X = R in place (L lower, n x n; R n x m): forward block substitution,
// the off-diagonal products on K1 (3M DMMA) reading the rows of L from
// Lh = L^H, the nb x nb diagonal solves by cuBLAS ZTRSM (~0.45 us per row:
// the latency of its sequential steps is the floor at n = 2048; a warp-per-
// column substitution kernel measured slower still).
int trsm_lower_k1(chfsi_ctx* ctx, int n, int m, const double2* L, long long ldl, const double2* Lh,
                  long long ldlh, double2* R, long long ldr) {
  const int nb = trsm_nb();
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
  for (int r0 = 0; r0 < n; r0 += nb) {
    const int rows = std::min(nb, n - r0);
    CK(k1_block_update(ctx, n, m, Lh, ldlh, r0, rows, 0, r0, R, ldr));
    CK_BLAS(cublasZtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N,
                        CUBLAS_DIAG_NON_UNIT, rows, m, &one,
                        reinterpret_cast<const cuDoubleComplex*>(L + r0 + (long long)r0 * ldl), (int)ldl,
                        reinterpret_cast<cuDoubleComplex*>(R + r0), (int)ldr));
  }
  return CHFSI_OK;
}

// L^H X = Y in place (backward block substitution; the rows of L^H are the
// conjugated columns of L, read by K1 directly from L's storage).
int trsm_lower_h_k1(chfsi_ctx* ctx, int n, int m, const double2* L, long long ldl, double2* Y,
                    long long ldy) {
  const int nb = trsm_nb();
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
  const int nblk = (n + nb - 1) / nb;
  for (int b = nblk - 1; b >= 0; --b) {
    const int r0 = b * nb, rows = std::min(nb, n - r0), k0 = r0 + rows;
    CK(k1_block_update(ctx, n, m, L, ldl, r0, rows, k0, n - k0, Y, ldy));
    CK_BLAS(cublasZtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C,
                        CUBLAS_DIAG_NON_UNIT, rows, m, &one,
                        reinterpret_cast<const cuDoubleComplex*>(L + r0 + (long long)r0 * ldl), (int)ldl,
                        reinterpret_cast<cuDoubleComplex*>(Y + r0), (int)ldy));
  }
  return CHFSI_OK;
}

}  // namespace

extern "C" {

int chfsi_heev_rr_z(chfsi_ctx* ctx, int n, void* A, long long lda, double* w, double tol,
                    int* used_fast) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(used_fast, "used_fast is NULL");
  *used_fast = 0;
  if (n == 0) return CHFSI_OK;
  CK_ARG(A && w && lda >= n, "bad argument");
  if (tol > 0.0 && n > 1) {
    bool done = false;
    CK(heev_near_diag(ctx, n, static_cast<double2*>(A), lda, w, tol, &done));
    if (done) {
      *used_fast = 1;
      return CHFSI_OK;
    }
  }
  return chfsi_heevd_z(ctx, n, A, lda, w);
}

int chfsi_heevd_z(chfsi_ctx* ctx, int n, void* A, long long lda, double* w) {
  CK_ARG(ctx, "ctx is NULL");
  if (n == 0) return CHFSI_OK;
  CK_ARG(A && w && lda >= n, "bad argument");
  int lwork = 0;
  cuDoubleComplex* a = static_cast<cuDoubleComplex*>(A);
  CK_SOLVER(cusolverDnZheevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR,
                                        CUBLAS_FILL_MODE_LOWER, n, a, (int)lda, w, &lwork));
  CK(ensure_ws(ctx, (size_t)lwork * sizeof(cuDoubleComplex)));
  CK_SOLVER(cusolverDnZheevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, a,
                             (int)lda, w, static_cast<cuDoubleComplex*>(ctx->ws), lwork,
                             ctx->dinfo));
  int info = 0;
  CK_CUDA(cudaMemcpyAsync(&info, ctx->dinfo, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info != 0) return fail(CHFSI_EEIG, "zheevd failed to converge, info=" + std::to_string(info));
  return CHFSI_OK;
}

int chfsi_colnorm_residual_sq_z(chfsi_ctx* ctx, int n, int w, const void* HP, long long ldhp,
                                const void* P, long long ldp, const double* lambda, double* res) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(HP && res, "NULL argument");
  CK_CUDA(chfsi::colnorm_residual_launch(static_cast<const double2*>(HP), ldhp,
                                         static_cast<const double2*>(P), ldp, lambda, n, w, res,
                                         ctx->stream, true));
  return CHFSI_OK;
}

int chfsi_colnorm_residual_z(chfsi_ctx* ctx, int n, int w, const void* HP, long long ldhp,
                             const void* P, long long ldp, const double* lambda, double* res) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(HP && res, "NULL argument");
  CK_CUDA(chfsi::colnorm_residual_launch(static_cast<const double2*>(HP), ldhp,
                                         static_cast<const double2*>(P), ldp, lambda, n, w, res,
                                         ctx->stream));
  return CHFSI_OK;
}

// ------------------------------------------------------------------- K5 ---

int chfsi_symmetrize_z(chfsi_ctx* ctx, int n, void* A, long long lda) {
  CK_ARG(ctx, "ctx is NULL");
  CK_CUDA(chfsi::symmetrize_launch(static_cast<double2*>(A), lda, n, ctx->stream));
  return CHFSI_OK;
}

int chfsi_herm_defect_z(chfsi_ctx* ctx, int n, const void* A, long long lda, double* defect,
                        double* maxabs) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(defect && maxabs, "NULL output");
  double* out = ctx->scalars + 4;
  CK_CUDA(chfsi::herm_defect_launch(static_cast<const double2*>(A), lda, n, out, ctx->stream));
  double h[2];
  CK_CUDA(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK_CUDA(cudaStreamSynchronize(ctx->stream));
  *defect = h[0];
  *maxabs = h[1];
  return CHFSI_OK;
}

int chfsi_conj_z(chfsi_ctx* ctx, int m, int n, void* A, long long lda) {
  CK_ARG(ctx, "ctx is NULL");
  CK_CUDA(chfsi::conj_inplace_launch(static_cast<double2*>(A), lda, m, n, ctx->stream));
  return CHFSI_OK;
}

int chfsi_potrf_z(chfsi_ctx* ctx, int n, void* A, long long lda, int* info) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(info, "info is NULL");
  *info = 0;
  if (n == 0) return CHFSI_OK;
  cuDoubleComplex* a = static_cast<cuDoubleComplex*>(A);
  int lwork = 0;
  CK_SOLVER(cusolverDnZpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, a, (int)lda, &lwork));
  CK(ensure_ws(ctx, (size_t)lwork * sizeof(cuDoubleComplex)));
  CK_SOLVER(cusolverDnZpotrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, a, (int)lda,
                             static_cast<cuDoubleComplex*>(ctx->ws), lwork, ctx->dinfo));
  CK_CUDA(cudaMemcpyAsync(info, ctx->dinfo, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (*info != 0)
    return fail(CHFSI_ENOTPD, "Cholesky pivot " + std::to_string(*info) + " is not positive");
  CK_CUDA(chfsi::zero_upper_launch(static_cast<double2*>(A), lda, n, ctx->stream));
  return CHFSI_OK;
}

int chfsi_trsm_z(chfsi_ctx* ctx, char side, char trans, int m, int n, const void* L,
                 long long ldl, void* B, long long ldb) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(side == 'L' || side == 'R', "side must be 'L' or 'R'");
  CK_ARG(trans == 'N' || trans == 'C', "trans must be 'N' or 'C'");
  if (m == 0 || n == 0) return CHFSI_OK;
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
  CK_BLAS(cublasZtrsm(ctx->blas, side == 'L' ? CUBLAS_SIDE_LEFT : CUBLAS_SIDE_RIGHT,
                      CUBLAS_FILL_MODE_LOWER, op_of(trans), CUBLAS_DIAG_NON_UNIT, m, n, &one,
                      static_cast<const cuDoubleComplex*>(L), (int)ldl,
                      static_cast<cuDoubleComplex*>(B), (int)ldb));
  return CHFSI_OK;
}

int chfsi_to_standard_async_z(chfsi_ctx* ctx, int n, void* A, long long lda, void* B,
                              long long ldb, int rowmajor_in, int* info_host) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(info_host, "info_host is NULL");
  if (n == 0) {
    *info_host = 0;
    return CHFSI_OK;
  }
  cudaStream_t s = ctx->stream;
  if (rowmajor_in) {
    CK(chfsi_conj_z(ctx, n, n, A, lda));
    CK(chfsi_conj_z(ctx, n, n, B, ldb));
  }
  cuDoubleComplex* b = static_cast<cuDoubleComplex*>(B);
  int lwork = 0;
  CK_SOLVER(cusolverDnZpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, b, (int)ldb, &lwork));
  CK(ensure_ws(ctx, (size_t)lwork * sizeof(cuDoubleComplex)));
  CK_SOLVER(cusolverDnZpotrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, b, (int)ldb,
                             static_cast<cuDoubleComplex*>(ctx->ws), lwork, ctx->dinfo));
  CK_CUDA(cudaMemcpyAsync(info_host, ctx->dinfo, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK_CUDA(chfsi::zero_upper_launch(static_cast<double2*>(B), ldb, n, s));
  CK(chfsi_trsm_z(ctx, 'L', 'N', n, n, B, ldb, A, lda));
  CK(chfsi_trsm_z(ctx, 'R', 'C', n, n, B, ldb, A, lda));
  CK(chfsi_symmetrize_z(ctx, n, A, lda));
  return CHFSI_OK;
}

int chfsi_to_standard_k1_z(chfsi_ctx* ctx, int n, void* A, long long lda, void* B, long long ldb,
                           int rowmajor_in, void* work, int* info_host) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(info_host, "info_host is NULL");
  CK_ARG(n == 0 || work, "work is NULL");
  if (n == 0) {
    *info_host = 0;
    return CHFSI_OK;
  }
  cudaStream_t s = ctx->stream;
  if (rowmajor_in) {
    CK(chfsi_conj_z(ctx, n, n, A, lda));
    CK(chfsi_conj_z(ctx, n, n, B, ldb));
  }
  cuDoubleComplex* b = static_cast<cuDoubleComplex*>(B);
  int lwork = 0;
  CK_SOLVER(cusolverDnZpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, b, (int)ldb, &lwork));
  CK(ensure_ws(ctx, (size_t)lwork * sizeof(cuDoubleComplex)));
  CK_SOLVER(cusolverDnZpotrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, b, (int)ldb,
                             static_cast<cuDoubleComplex*>(ctx->ws), lwork, ctx->dinfo));
  CK_CUDA(cudaMemcpyAsync(info_host, ctx->dinfo, sizeof(int), cudaMemcpyDeviceToHost, s));
  double2* l = static_cast<double2*>(B);
  double2* a = static_cast<double2*>(A);
  double2* lh = static_cast<double2*>(work);  // L^H (n x n, ld n)
  double2* t = lh + (size_t)n * n;            // Z^H, then H (n x n, ld n)
  CK_CUDA(chfsi::zero_upper_launch(l, ldb, n, s));
  CK_CUDA(chfsi::conj_transpose_launch(l, ldb, lh, n, n, s));
  CK(trsm_lower_k1(ctx, n, n, l, ldb, lh, n, a, lda));  // Z = L^-1 A
  CK_CUDA(chfsi::conj_transpose_launch(a, lda, t, n, n, s));
  CK(trsm_lower_k1(ctx, n, n, l, ldb, lh, n, t, n));    // H = L^-1 Z^H (= Z L^-H, Hermitian)
  CK_CUDA(cudaMemcpy2DAsync(a, (size_t)lda * sizeof(double2), t, (size_t)n * sizeof(double2),
                            (size_t)n * sizeof(double2), n, cudaMemcpyDeviceToDevice, s));
  CK(chfsi_symmetrize_z(ctx, n, A, lda));
  return CHFSI_OK;
}

int chfsi_herm_defect_async_z(chfsi_ctx* ctx, int n, const void* A, long long lda,
                              double* out_host) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(out_host, "NULL output");
  if (n == 0) {
    out_host[0] = out_host[1] = 0.0;
    return CHFSI_OK;
  }
  double* out = ctx->scalars + 4;
  CK_CUDA(chfsi::herm_defect_launch(static_cast<const double2*>(A), lda, n, out, ctx->stream));
  CK_CUDA(cudaMemcpyAsync(out_host, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  return CHFSI_OK;
}

int chfsi_to_standard_z(chfsi_ctx* ctx, int n, void* A, long long lda, void* B, long long ldb,
                        int rowmajor_in, int* info) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(info, "info is NULL");
  if (rowmajor_in) {  // Hermitian: row-major bytes == conj of the column-major matrix
    CK(chfsi_conj_z(ctx, n, n, A, lda));
    CK(chfsi_conj_z(ctx, n, n, B, ldb));
  }
  CK(chfsi_potrf_z(ctx, n, B, ldb, info));                  // B = L L^H
  CK(chfsi_trsm_z(ctx, 'L', 'N', n, n, B, ldb, A, lda));    // Z = L^-1 A
  CK(chfsi_trsm_z(ctx, 'R', 'C', n, n, B, ldb, A, lda));    // H = Z L^-H
  CK(chfsi_symmetrize_z(ctx, n, A, lda));                   // (H + H^H)/2
  return CHFSI_OK;
}

int chfsi_back_transform_z(chfsi_ctx* ctx, int n, int nev, const void* L, long long ldl, void* Y,
                           long long ldy) {
  // Y <- L^-H Y by backward block substitution: per block of rows the
  // product with the rows of L^H right of the diagonal on K1 (3M DMMA,
  // reading L's own columns conjugated), then a small ZTRSM on the diagonal
  // block. cuBLAS's single ZTRSM of the whole triangle was 1.07 ms at
  // n = 2048, nev = 128 (latency of its sequential blocks).
  CK_ARG(ctx, "ctx is NULL");
  if (n == 0 || nev == 0) return CHFSI_OK;
  return trsm_lower_h_k1(ctx, n, nev, static_cast<const double2*>(L), ldl, static_cast<double2*>(Y),
                         ldy);
}

}  // extern "C"
