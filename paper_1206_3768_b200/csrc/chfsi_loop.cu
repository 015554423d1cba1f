// Native ChFSI inner loop (chfsi_solve_loop_z, include/chfsi.h).
//
// Restates the pass structure of the reference solver loop
// (spectral_chain/chfsi.py:328-373) on top of libchfsi's own entry points:
//
//   filter (K1 x deg)                                   chfsi.py:331-334
//   2x CGS vs the locked block + QR, rank repair        chfsi.py:242-261
//   Rayleigh-Ritz on the panel, residual norms          chfsi.py:337-350
//   lock the leading Ritz pairs with res < tol          chfsi.py:352-366
//   refresh the window [ritz[n_lock], ritz[-1]]         chfsi.py:367-373
//
// Host work per pass is a few dozen scalar operations; the only host<->device
// traffic is the blk Ritz values and residuals the locking test needs (one
// stream synchronisation per pass, plus the near-diagonal eigensolver's
// regime checks). Device phase times are taken with events on the stream.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <utility>
#include <cmath>
#include <vector>

#include "abi_internal.h"

namespace {

using chfsi::fail;

// chfsi.py:264-271: clamp the refreshed window back to scale_ref < a < b.
void safe_window(double scale_ref, double a, double b, double* out_a, double* out_b) {
  if (!std::isfinite(scale_ref) || !std::isfinite(a) || !std::isfinite(b) || !(scale_ref < b)) {
    *out_a = scale_ref + 0.5;
    *out_b = scale_ref + 1.0;
    return;
  }
  if (!(scale_ref < a && a < b)) a = scale_ref + 0.5 * (b - scale_ref);
  *out_a = a;
  *out_b = b;
}

// Per-vector degree (oracle/chfsi_oracle.py adaptive_degree
// restates it with the same C-library operations): damp the residual r of a
// Ritz pair at lambda to tol under the window (a, b).
constexpr int kAdaptiveMargin = 2;  // oracle ADAPTIVE_MARGIN
int adaptive_degree(double lam, double r, double a, double b, double tol, int d_min, int d_max) {
  if (std::isnan(r) || std::isnan(lam)) return d_max;
  if (!(r > tol)) return d_min;
  const double c = (a + b) / 2, e = (b - a) / 2;
  const double t = (lam - c) / e;
  if (!(t < -1.0)) return d_max;
  const double rho = -t + std::sqrt(t * t - 1.0);
  const double d = std::ceil(std::log(r / tol) / std::log(rho)) + kAdaptiveMargin;
  if (!(d < (double)d_max)) return d_max;  // also catches inf / nan
  return d < (double)d_min ? d_min : (int)d;
}

double2* col(void* base, long long ld, int j) { return static_cast<double2*>(base) + (long long)j * ld; }

int ensure_events(chfsi_ctx* ctx) {
  for (cudaEvent_t& e : ctx->loop_ev)
    if (!e) CK_CUDA(cudaEventCreate(&e));
  return CHFSI_OK;
}

// CHFSI_ROTATE_PAIR=0: the two Rayleigh-Ritz rotations as separate ZGEMMs (A/B)
bool rotate_pair_off() {
  static const bool off = [] {
    const char* e = getenv("CHFSI_ROTATE_PAIR");
    return e && atoi(e) == 0;
  }();
  return off;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  return cudaEventElapsedTime(&ms, a, b) == cudaSuccess ? ms : 0.f;
}

// CHFSI_QR_DEFER=0: the Cholesky-QR acceptance test synchronises inside
// the QR (one host round trip per pass more) instead of at the pass's end
bool qr_defer_enabled() {
  static const bool on = [] {
    const char* e = getenv("CHFSI_QR_DEFER");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// Two CGS passes against the locked block, then QR; rank-deficient columns
// are replaced through the fill callback and the whole panel is redone,
// at most `retries` times (chfsi.py:242-261).
//   mode 1 (speculative): CGS + Cholesky-QR2 with the acceptance test
//          deferred to the pass's own synchronisation (no host round trip);
//   mode 2: after a rejected speculation — the pre-QR panel (already
//          projected) is restored and the full QR path runs.
int orthonormalize(chfsi_ctx* ctx, chfsi_loop* L, void* work, int width, int mode = 0) {
  const int n = L->n;
  constexpr int retries = 3;
  if (mode == 1) {
    if (L->nlocked)
      CK(chfsi_cgs_project_z(ctx, n, L->nlocked, width, L->locked, n, work, n, L->coef));
    return chfsi::qr_orthonormalize_deferred(ctx, n, width, work, n);
  }
  if (mode == 2) CK(chfsi::qr_deferred_restore(ctx, n, width, work));
  std::vector<int> dead(width);
  for (int attempt = 0;; ++attempt) {
    if (L->nlocked && !(mode == 2 && attempt == 0))
      CK(chfsi_cgs_project_z(ctx, n, L->nlocked, width, L->locked, n, work, n, L->coef));
    int ndead = 0;
    const int rc = chfsi_qr_orthonormalize_z(ctx, n, width, work, n, dead.data(), &ndead);
    if (rc != CHFSI_ERANK) return rc;
    if (attempt == retries || !L->fill) return rc;
    if (L->fill(L->user, work, n, n, dead.data(), ndead) != 0)
      return fail(CHFSI_EINVAL, "rank-repair fill callback failed");
  }
}

// HP = H P; G = P^H HP symmetrised; eigenpairs (near-diagonal solver when
// allowed, else zheevd); P W, HP W; residual norms (chfsi.py:337-350).
// P_rot = Q W and HP_rot = HP W (n x w each, ld n) as ONE strided-batched
// ZGEMM (batch 2, W shared) when the two pairs of blocks are equally ordered
// in memory (the batch strides must be non-negative); two ZGEMMs otherwise.
int rotate_pair(chfsi_ctx* ctx, int n, int w, const void* q, const void* hp, const void* W,
                long long ldw, void* rot_p, void* hp_rot) {
  const auto* a0 = static_cast<const cuDoubleComplex*>(q);
  const auto* a1 = static_cast<const cuDoubleComplex*>(hp);
  auto* c0 = static_cast<cuDoubleComplex*>(rot_p);
  auto* c1 = static_cast<cuDoubleComplex*>(hp_rot);
  if ((a1 < a0) != (c1 < c0) || rotate_pair_off()) {
    CK(chfsi_gemm_z(ctx, 'N', 'N', n, w, w, 1.0, 0.0, q, n, W, ldw, 0.0, 0.0, rot_p, n));
    return chfsi_gemm_z(ctx, 'N', 'N', n, w, w, 1.0, 0.0, hp, n, W, ldw, 0.0, 0.0, hp_rot, n);
  }
  if (a1 < a0) {
    std::swap(a0, a1);
    std::swap(c0, c1);
  }
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  CK_BLAS(cublasZgemmStridedBatched(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_N, n, w, w, &one, a0, n,
                                    (long long)(a1 - a0), static_cast<const cuDoubleComplex*>(W),
                                    (int)ldw, 0, &zero, c0, n, (long long)(c1 - c0), 2));
  return CHFSI_OK;
}

// CHFSI_RR_DEFER=0: the near-diagonal eigensolver's verdict is awaited inside
// Rayleigh-Ritz (one host round trip per pass more) instead of at the pass's end
bool rr_defer_enabled() {
  static const bool on = [] {
    const char* e = getenv("CHFSI_RR_DEFER");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// `speculate`: the near-diagonal eigensolver is queued without waiting for
// its verdict and the rotations / residual norms follow at once (*pending =
// true: the caller judges it after the pass's synchronisation and calls
// rayleigh_ritz_redo when it failed). Measured before: the verdict's round
// trip left the stream idle 26-41 us per pass until the rotation started.
int rayleigh_ritz(chfsi_ctx* ctx, chfsi_loop* L, const void* q, void* rot_p, int width, double eig_tol,
                  int* used_fast, bool speculate = false, bool* pending = nullptr) {
  const int n = L->n;
  const long long ldg = L->blk;
  if (pending) *pending = false;
  CK(chfsi_cheb_step_z(ctx, n, width, L->H, L->ldh, L->conj_h, q, n, nullptr, 0, L->hp, n, 1.0, 0.0,
                       0.0));
  CK(chfsi_gemm_z(ctx, 'C', 'N', width, width, n, 1.0, 0.0, q, n, L->hp, n, 0.0, 0.0, L->g, ldg));
  CK(chfsi_symmetrize_z(ctx, width, L->g, ldg));
  bool queued = false;
  if (speculate && pending)
    CK(chfsi::heev_rr_speculative(ctx, width, L->g, ldg, L->ritz_d, eig_tol, &queued));
  if (queued) *pending = true;
  else CK(chfsi_heev_rr_z(ctx, width, L->g, ldg, L->ritz_d, eig_tol, used_fast));
  CK(rotate_pair(ctx, n, width, q, L->hp, L->g, ldg, rot_p, L->hp_rot));
  CK(chfsi_colnorm_residual_z(ctx, n, width, L->hp_rot, n, rot_p, n, L->ritz_d, L->res_d));
  return CHFSI_OK;
}

// The speculative eigensolver failed (G is untouched, H P is still in L->hp):
// zheevd, then the rotations and residual norms again.
int rayleigh_ritz_redo(chfsi_ctx* ctx, chfsi_loop* L, const void* q, void* rot_p, int width) {
  const int n = L->n;
  const long long ldg = L->blk;
  CK(chfsi_heevd_z(ctx, width, L->g, ldg, L->ritz_d));
  CK(rotate_pair(ctx, n, width, q, L->hp, L->g, ldg, rot_p, L->hp_rot));
  CK(chfsi_colnorm_residual_z(ctx, n, width, L->hp_rot, n, rot_p, n, L->ritz_d, L->res_d));
  return CHFSI_OK;
}

// ------------------------------------------------ row-sharded (multi-GPU) ---
// Every n x w block holds this rank's n_local rows (ld n_local). Products
// that contract over rows leave partial w x w / w-sized results, summed over
// the ranks by the allreduce callback (NCCL returns identical bytes on all
// ranks, so the replicated factorizations and decisions stay consistent).

int allreduce(chfsi_loop* L, void* buf, long long count) {
  if (L->allreduce(L->user, buf, count) != 0) return fail(CHFSI_ENCCL, "allreduce callback failed");
  return CHFSI_OK;
}

// diag(A)[0..w) of a device w x w block (ld lda) -> host (real parts), synchronous
int read_diag_re(chfsi_ctx* ctx, const void* A, long long lda, int w, double* out) {
  CK(chfsi::ensure_pinned(ctx, (size_t)w * sizeof(double2)));
  double2* h = static_cast<double2*>(ctx->pinned);
  CK_CUDA(cudaMemcpy2DAsync(h, sizeof(double2), A, (size_t)(lda + 1) * sizeof(double2),
                            sizeof(double2), w, cudaMemcpyDeviceToHost, ctx->stream));
  CK_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < w; ++i) out[i] = h[i].x;
  return CHFSI_OK;
}

// Two CGS passes + Cholesky-QR2 on local rows with all-reduced Grams; the
// rank test and any failure fall back to the full-matrix QR (gather, then
// chfsi_qr_orthonormalize_z replicated on every rank, local rows kept).
int orthonormalize_dist(chfsi_ctx* ctx, chfsi_loop* L, void* work, int width) {
  const int n = L->n, nl = L->n_local, nk = L->nlocked;
  constexpr int retries = 3;
  std::vector<int> dead(width);
  std::vector<double> d0(width), r1(width), r2(width);
  for (int attempt = 0;; ++attempt) {
    for (int pass = 0; nk && pass < 2; ++pass) {  // coef = L^H W summed; W -= L coef
      CK(chfsi_gemm_z(ctx, 'C', 'N', nk, width, nl, 1.0, 0.0, L->locked, nl, work, nl, 0.0, 0.0,
                      L->coef, nk));
      CK(allreduce(L, L->coef, 2LL * nk * width));
      CK(chfsi_gemm_z(ctx, 'N', 'N', nl, width, nk, -1.0, 0.0, L->locked, nl, L->coef, nk, 1.0, 0.0,
                      work, nl));
    }
    // backup for the fallback: hp_rot is free until Rayleigh-Ritz
    CK_CUDA(cudaMemcpyAsync(L->hp_rot, work, (size_t)nl * width * sizeof(double2),
                            cudaMemcpyDeviceToDevice, ctx->stream));
    bool ok = true;
    double fro2 = 0.0;
    for (int pass = 0; ok && pass < 2; ++pass) {
      CK(chfsi_gemm_z(ctx, 'C', 'N', width, width, nl, 1.0, 0.0, work, nl, work, nl, 0.0, 0.0, L->g,
                      width));
      CK(allreduce(L, L->g, 2LL * width * width));
      if (pass == 0) {
        CK(read_diag_re(ctx, L->g, width, width, d0.data()));
        for (int i = 0; i < width; ++i) fro2 += d0[i];
      }
      int info = 0;
      const int rc = chfsi_potrf_z(ctx, width, L->g, width, &info);  // G = R^H R, L = R^H
      if (rc == CHFSI_ENOTPD) {
        ok = false;
        break;
      }
      CK(rc);
      CK(read_diag_re(ctx, L->g, width, width, pass == 0 ? r1.data() : r2.data()));
      CK(chfsi_trsm_z(ctx, 'R', 'C', nl, width, L->g, width, work, nl));  // W <- W R^-1
    }
    if (ok) {  // same acceptance as chfsi_qr_orthonormalize_z's Cholesky-QR2
      const double fro = std::sqrt(fro2), safe = 1e-11 * fro;
      for (int i = 0; ok && i < width; ++i)
        ok = std::isfinite(fro) && r1[i] * r2[i] >= safe && std::fabs(r2[i] - 1.0) <= 1e-6;
      if (ok) return CHFSI_OK;
    }
    // fallback: the full-matrix QR, replicated
    CK_CUDA(cudaMemcpyAsync(work, L->hp_rot, (size_t)nl * width * sizeof(double2),
                            cudaMemcpyDeviceToDevice, ctx->stream));
    void* fullp = nullptr;
    if (!L->gather || L->gather(L->user, work, nl, width, &fullp) != 0 || !fullp)
      return fail(CHFSI_EINVAL, "gather callback failed");
    int ndead = 0;
    const int rc = chfsi_qr_orthonormalize_z(ctx, n, width, fullp, n, dead.data(), &ndead);
    if (rc == CHFSI_OK) {
      CK_CUDA(cudaMemcpy2DAsync(work, (size_t)nl * sizeof(double2),
                                static_cast<double2*>(fullp) + L->row0, (size_t)n * sizeof(double2),
                                (size_t)nl * sizeof(double2), width, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      return CHFSI_OK;
    }
    if (rc != CHFSI_ERANK) return rc;
    if (attempt == retries || !L->fill) return rc;
    if (L->fill(L->user, work, nl, nl, dead.data(), ndead) != 0)
      return fail(CHFSI_EINVAL, "rank-repair fill callback failed");
  }
}

// Rayleigh-Ritz on local rows: HP from the hp callback, G = P^H HP summed,
// replicated eigensolver, local rotations, residual squares summed.
int rayleigh_ritz_dist(chfsi_ctx* ctx, chfsi_loop* L, const void* q, void* rot_p, int width,
                       double eig_tol, int* used_fast) {
  const int nl = L->n_local;
  if (L->hp_fn(L->user, q, L->hp, nl, width) != 0) return fail(CHFSI_EINVAL, "hp callback failed");
  CK(chfsi_gemm_z(ctx, 'C', 'N', width, width, nl, 1.0, 0.0, q, nl, L->hp, nl, 0.0, 0.0, L->g, width));
  CK(allreduce(L, L->g, 2LL * width * width));
  CK(chfsi_symmetrize_z(ctx, width, L->g, width));
  CK(chfsi_heev_rr_z(ctx, width, L->g, width, L->ritz_d, eig_tol, used_fast));
  CK(chfsi_gemm_z(ctx, 'N', 'N', nl, width, width, 1.0, 0.0, q, nl, L->g, width, 0.0, 0.0, rot_p, nl));
  CK(chfsi_gemm_z(ctx, 'N', 'N', nl, width, width, 1.0, 0.0, L->hp, nl, L->g, width, 0.0, 0.0,
                  L->hp_rot, nl));
  CK(chfsi_colnorm_residual_sq_z(ctx, nl, width, L->hp_rot, nl, rot_p, nl, L->ritz_d, L->res_d));
  CK(allreduce(L, L->res_d, width));
  return CHFSI_OK;
}

}  // namespace

extern "C" int chfsi_solve_loop_z(chfsi_ctx* ctx, chfsi_loop* L) {
  CK_ARG(ctx && L, "NULL argument");
  CK_ARG(L->n >= 1 && 1 <= L->nev && L->nev <= L->blk && L->blk <= L->n, "need 1 <= nev <= blk <= n");
  CK_ARG(L->deg >= 1 && L->max_repeats >= 0 && L->tol > 0, "bad degree / repeats / tolerance");
  CK_ARG(L->H && L->bufs[0] && L->bufs[1] && L->hp && L->hp_rot && L->locked && L->g && L->coef &&
             L->ritz_d && L->res_d,
         "NULL device buffer");
  CK_ARG(L->locked_vals && L->locked_res && L->locked_per_loop && L->ritz && L->res,
         "NULL host output");
  CK_ARG(L->pb == 0 || L->pb == 1, "bad panel buffer index");
  CK_ARG(L->off >= 0 && L->width >= 1 && L->off + L->width <= L->blk, "bad panel window");
  const bool dist = L->allreduce != nullptr;
  CK_ARG(!dist || (L->hp_fn && L->filter && L->n_local >= 1 && L->row0 >= 0 &&
                   L->row0 + L->n_local <= L->n),
         "row-sharded loop needs filter and hp callbacks and a valid row range");
  CK(ensure_events(ctx));
  cudaStream_t s = ctx->stream;
  // phase timers: pass p records into event set p % 2; a pass's elapsed
  // times are read once the next pass's filter is queued (not inside the
  // device-idle gap after the per-pass sync)
  cudaEvent_t* ev = ctx->loop_ev;
  cudaEvent_t* pending = nullptr;
  auto read_timers = [&]() {
    if (!pending) return;
    L->t_filter += 1e-3 * elapsed(pending[0], pending[1]);
    L->t_ortho += 1e-3 * elapsed(pending[1], pending[2]);
    L->t_rr += 1e-3 * elapsed(pending[2], pending[3]);
    pending = nullptr;
  };
  const int n = L->n;
  const int nl = dist ? L->n_local : n;  // rows (and ld) of every n x w block here
  CK_ARG(!L->adaptive || (L->degs && L->perm_d && 1 <= L->deg_min && L->deg_min <= L->deg),
         "adaptive degree needs degs, perm_d and 1 <= deg_min <= deg");
  // pinned staging: [ritz | res] readback, then the adaptive column order
  CK(chfsi::ensure_pinned(ctx, 2 * (size_t)L->blk * sizeof(double) + (size_t)L->blk * sizeof(int)));
  // (ritz | res) readback: ONE copy when the two device arrays are the halves
  // of one 2 blk buffer (res_d == ritz_d + blk; the Python workspace), else two
  const bool packed = static_cast<double*>(L->res_d) == static_cast<double*>(L->ritz_d) + L->blk;
  auto readback = [&](double* host, int width) -> int {
    if (packed) {
      CK_CUDA(cudaMemcpyAsync(host, L->ritz_d, (size_t)(L->blk + width) * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
      return CHFSI_OK;
    }
    CK_CUDA(cudaMemcpyAsync(host, L->ritz_d, (size_t)width * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaMemcpyAsync(host + width, L->res_d, (size_t)width * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    return CHFSI_OK;
  };
  bool have_degs = false;
  std::vector<int> dtmp, order;
  // H * (next panel) from the previous pass's Rayleigh-Ritz: hp_rot columns
  // [n_lock, width) are H P_rot for exactly the columns the next panel keeps
  const bool reuse = L->reuse_hp && !dist && !L->filter;
  const void* hy_next = nullptr;  // H * (next panel): hp_rot columns, or hp after an adaptive gather
  bool hp_ready = false;

  while (L->inner_loops < L->max_repeats) {
    L->inner_loops += 1;
    const int width = L->width;
    void* panel = col(L->bufs[L->pb], nl, L->off);
    void* other = L->bufs[1 - L->pb];
    ev = ctx->loop_ev + 4 * (L->inner_loops & 1);

    // ---- filter (chfsi.py:331-334)
    CK_CUDA(cudaEventRecord(ev[0], s));
    void* result = nullptr;
    const int* degs = have_degs ? L->degs : nullptr;  // adaptive: sorted per-column degrees
    if (L->filter) {
      if (L->filter(L->user, panel, other, nl, width, L->deg, degs, L->win_a, L->win_b,
                    L->win_scale_ref, &result) != 0 || !result)
        return fail(CHFSI_EINVAL, "filter callback failed");
    } else if (degs) {
      const void* hy0 = hp_ready ? hy_next : nullptr;
      CK(chfsi::filter_degrees_impl(ctx, n, width, L->H, L->ldh, L->conj_h, panel, n, hy0, n, other,
                                    panel, n, degs, L->win_a, L->win_b, L->win_scale_ref, &result));
      if (hy0) {
        L->filter_k1_launches -= 1;
        L->filter_k1_flops -= 8.0 * (double)n * (double)n * (double)width;
      }
    } else {
      const void* hy0 = hp_ready ? hy_next : nullptr;
      CK(chfsi::filter_z_impl(ctx, n, width, L->H, L->ldh, L->conj_h, panel, n, hy0, n, other, panel,
                              n, L->deg, L->win_a, L->win_b, L->win_scale_ref, &result));
      if (hy0) {  // one elementwise step instead of a K1 product
        L->filter_k1_launches -= 1;
        L->filter_k1_flops -= 8.0 * (double)n * (double)n * (double)width;
      }
    }
    hp_ready = false;
    CK_CUDA(cudaEventRecord(ev[1], s));
    read_timers();  // the previous pass's (its events completed at its sync)
    long long dsum = (long long)L->deg * width;
    if (degs) {
      dsum = 0;
      for (int j = 0; j < width; ++j) dsum += degs[j];
    }
    L->filter_launches += degs ? degs[width - 1] : L->deg;
    L->filtered_vectors += width;
    L->matvecs += dsum;
    L->filter_degree_sum += dsum;
    L->filter_flops += 8.0 * (double)n * (double)n * (double)dsum;
    L->filter_k1_launches += degs ? degs[width - 1] : L->deg;
    L->filter_k1_flops += 8.0 * (double)n * (double)n * (double)dsum;
    const bool q_in_other = result == other;

    // ---- orthonormalize (chfsi.py:335-336); single-GPU: Cholesky-QR2 with
    // its acceptance test judged after this pass's readback (speculative)
    const bool spec = !dist && qr_defer_enabled() && ctx->qr_mode == 0 && ctx->qr_linear2;
    CK(dist ? orthonormalize_dist(ctx, L, result, width)
            : orthonormalize(ctx, L, result, width, spec ? 1 : 0));
    CK_CUDA(cudaEventRecord(ev[2], s));

    // ---- Rayleigh-Ritz into the buffer the filter left free (chfsi.py:337-350)
    const int rot_pb = q_in_other ? L->pb : 1 - L->pb;
    void* rot_p = L->bufs[rot_pb];
    // The near-diagonal eigensolver is tried on every pass: when G is not in
    // its regime it bails out after one O(w^2) measurement (~30 us), and
    // zheevd runs instead (measured: 4 zheevd calls less per warm C2 problem).
    const double eig_tol = L->rr_fast_tol > 0.0 ? L->rr_fast_tol : 0.0;
    int used_fast = 0;
    bool spec_redo = false;  // the speculative QR must be judged (and redone) now
    bool nd_pending = false; // the near-diagonal eigensolver's verdict is still out
    if (dist) {
      CK(rayleigh_ritz_dist(ctx, L, result, rot_p, width, eig_tol, &used_fast));
    } else {
      const int rc = rayleigh_ritz(ctx, L, result, rot_p, width, eig_tol, &used_fast,
                                   rr_defer_enabled(), &nd_pending);
      if (rc != CHFSI_OK) {
        // A failed Cholesky inside the speculative QR leaves non-finite
        // panels; the eigensolver then fails before the pass's readback.
        // Judge the QR first: a rejection redoes the pass below; an
        // accepted QR means the failure is genuine.
        if (!spec) return rc;
        CK_CUDA(cudaStreamSynchronize(s));
        bool accept = true;
        CK(chfsi::qr_deferred_verdict(ctx, &accept));
        if (accept) return rc;
        spec_redo = true;
        used_fast = 0;
      }
    }
    CK_CUDA(cudaEventRecord(ev[3], s));
    L->rr_fast_eigs += used_fast;
    L->residual_check_matvecs += width;
    L->matvecs += width;
    double* host = static_cast<double*>(ctx->pinned);  // (re-read: RR may have grown it)
    CK(readback(host, width));
    CK_CUDA(cudaStreamSynchronize(s));
    if (spec) {  // the speculative QR's acceptance test (its inputs are on the host now)
      bool accept = false;
      if (!spec_redo) CK(chfsi::qr_deferred_verdict(ctx, &accept));
      if (!accept) {  // rare: redo the pass's QR and Rayleigh-Ritz on the full path
        if (nd_pending) {  // (its input came from the rejected QR: the verdict is moot)
          bool ignored = false;
          CK(chfsi::heev_rr_verdict(ctx, &ignored));
          nd_pending = false;
        }
        CK(orthonormalize(ctx, L, result, width, 2));
        L->rr_fast_eigs -= used_fast;
        used_fast = 0;
        CK(rayleigh_ritz(ctx, L, result, rot_p, width, eig_tol, &used_fast));
        L->rr_fast_eigs += used_fast;
        host = static_cast<double*>(ctx->pinned);
        CK(readback(host, width));
        CK_CUDA(cudaStreamSynchronize(s));
        L->qr_redone += 1;
      }
    }
    if (nd_pending) {  // the speculative eigensolver's verdict (its status is on the host now)
      bool done = false;
      CK(chfsi::heev_rr_verdict(ctx, &done));
      if (done) {
        L->rr_fast_eigs += 1;
      } else {  // not near-diagonal: zheevd, rotations and residuals again
        const auto t_redo = std::chrono::steady_clock::now();
        CK(rayleigh_ritz_redo(ctx, L, result, rot_p, width));
        host = static_cast<double*>(ctx->pinned);
        CK(readback(host, width));
        CK_CUDA(cudaStreamSynchronize(s));
        // (behind the pass's event set: the stream was idle at the start, so wall time = device time)
        L->t_rr += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_redo).count();
      }
    }
    pending = ev;
    double* hres = host + (packed ? L->blk : width);
    if (dist)  // summed squares of the local row norms
      for (int j = 0; j < width; ++j) hres[j] = std::sqrt(hres[j]);
    const double* ritz = host;
    const double* res = hres;
    for (int j = 0; j < width; ++j) {
      L->ritz[j] = ritz[j];
      L->res[j] = res[j];
    }

    // ---- locking (chfsi.py:352-366)
    int n_lock = 0;
    while (n_lock < width && L->nlocked + n_lock < L->nev && res[n_lock] < L->tol) ++n_lock;
    if (n_lock) {
      for (int j = 0; j < n_lock; ++j) {
        L->locked_vals[L->nlocked + j] = ritz[j];
        L->locked_res[L->nlocked + j] = res[j];
      }
      CK_CUDA(cudaMemcpyAsync(col(L->locked, nl, L->nlocked), rot_p,
                              (size_t)nl * n_lock * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      L->nlocked += n_lock;
    }
    L->locked_per_loop[L->inner_loops - 1] = n_lock;
    L->last_rot_pb = rot_pb;
    L->last_width = width;
    L->last_nlock = n_lock;
    if (L->nlocked >= L->nev) {
      L->converged = 1;
      break;
    }

    // ---- next panel and window (chfsi.py:367-373)
    hp_ready = reuse;  // hp_rot[:, n_lock:width] = H * the next panel
    hy_next = col(L->hp_rot, nl, n_lock);
    L->pb = rot_pb;
    L->off = n_lock;
    L->width = width - n_lock;
    L->win_scale_ref = ritz[n_lock];
    safe_window(ritz[n_lock], ritz[width - 1], L->win_b, &L->win_a, &L->win_b);

    // ---- adaptive: per-vector degrees for the next panel, columns sorted
    // by ascending degree (stable), gathered into the other buffer
    if (L->adaptive) {
      const int wn = L->width;
      dtmp.resize(wn);
      order.resize(wn);
      for (int i = 0; i < wn; ++i) {
        dtmp[i] = adaptive_degree(ritz[n_lock + i], res[n_lock + i], L->win_a, L->win_b, L->tol,
                                  L->deg_min, L->deg);
        order[i] = i;
      }
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return dtmp[x] < dtmp[y]; });
      bool ident = true;
      for (int i = 0; i < wn; ++i) {
        L->degs[i] = dtmp[order[i]];
        ident = ident && order[i] == i;
      }
      if (!ident) {
        int* hperm = reinterpret_cast<int*>(static_cast<double*>(ctx->pinned) + 2 * (size_t)L->blk);
        for (int i = 0; i < wn; ++i) hperm[i] = order[i];
        CK_CUDA(cudaMemcpyAsync(L->perm_d, hperm, (size_t)wn * sizeof(int), cudaMemcpyHostToDevice, s));
        CK_CUDA(chfsi::nd_gather_cols_launch(col(L->bufs[L->pb], nl, L->off), nl, nl, wn, L->perm_d,
                                             static_cast<double2*>(L->bufs[1 - L->pb]), nl, s));
        if (hp_ready) {  // H * panel in the same column order (hp is free until Rayleigh-Ritz)
          CK_CUDA(chfsi::nd_gather_cols_launch(static_cast<const double2*>(hy_next), nl, nl, wn,
                                               L->perm_d, static_cast<double2*>(L->hp), nl, s));
          hy_next = L->hp;
        }
        L->pb = 1 - L->pb;
        L->off = 0;
      }
      have_degs = true;
    }
  }
  read_timers();
  // chained-mode tail: [locked | unlocked remainder of the final panel]
  if (L->tail && L->inner_loops > 0) {
    const size_t col_bytes = (size_t)nl * sizeof(double2);
    if (L->nlocked)
      CK_CUDA(cudaMemcpyAsync(L->tail, L->locked, col_bytes * L->nlocked, cudaMemcpyDeviceToDevice, s));
    const int rest = L->last_width - L->last_nlock;
    if (rest > 0)
      CK_CUDA(cudaMemcpyAsync(col(L->tail, nl, L->nlocked),
                              col(L->bufs[L->last_rot_pb], nl, L->last_nlock), col_bytes * rest,
                              cudaMemcpyDeviceToDevice, s));
  }
  return CHFSI_OK;
}

// ------------------------------------------------------ row-sharded Lanczos ---
// The k-step Lanczos chain (chfsi.py:125-162) with H, the basis and every
// n-vector split by rows: per step the GEMV runs on this rank's rows of H
// against the gathered full vector, and alpha, the reorthogonalisation
// coefficients and ||r||^2 are partial sums completed by the allreduce
// callback. The multi-kernel path of chfsi_lanczos_z on local rows, with the
// same breakdown rule (device flag; every rank sees the same beta).

extern "C" long long chfsi_lanczos_rows_ws_bytes(int n_local, int k) {
  // u, r (n_local each), coef (k complex), alphas, betas (k), nrm (1), padding
  return 2LL * n_local * sizeof(double2) + (long long)k * sizeof(double2) +
         (2LL * k + 8) * sizeof(double) + 256;
}

extern "C" int chfsi_lanczos_rows_z(chfsi_ctx* ctx, int n, int k, const void* H_rows, long long ldh,
                                    int conj_h, int row0, int n_local, const void* q0, void* V_local,
                                    void* ws, chfsi_allreduce_cb allreduce_fn, chfsi_gather_cb gather_fn,
                                    void* user, double* alphas, double* betas, double* beta_last,
                                    int* steps) {
  CK_ARG(ctx, "ctx is NULL");
  CK_ARG(n >= 1 && k >= 1 && k <= n, "need 1 <= k <= n");
  CK_ARG(n_local >= 1 && row0 >= 0 && row0 + n_local <= n, "bad row range");
  CK_ARG(H_rows && q0 && V_local && ws && allreduce_fn && gather_fn && alphas && betas && beta_last &&
             steps,
         "NULL argument");
  cudaStream_t s = ctx->stream;
  const int nl = n_local;
  char* base = static_cast<char*>(ws);
  double2* u = reinterpret_cast<double2*>(base);
  double2* r = u + nl;
  double2* coef = r + nl;
  double* al_d = reinterpret_cast<double*>(coef + k);
  double* be_d = al_d + k;
  double* nrm = be_d + k;
  double2* V = static_cast<double2*>(V_local);
  const double2* hh = static_cast<const double2*>(H_rows);
  chfsi::LanczosState* st = ctx->lstate;
  const int* done = &st->done;
  auto reduce = [&](void* buf, long long count) -> int {
    if (allreduce_fn(user, buf, count) != 0) return fail(CHFSI_ENCCL, "allreduce callback failed");
    return CHFSI_OK;
  };
  CK_CUDA(cudaMemsetAsync(st, 0, sizeof(chfsi::LanczosState), s));
  CK_CUDA(cudaMemsetAsync(be_d, 0, (size_t)k * sizeof(double), s));
  // q = q0 / ||q0|| on the full (replicated) vector, then this rank's rows
  CK_CUDA(chfsi::norm2_launch(static_cast<const double2*>(q0), n, ctx->partial, nrm, nullptr, s));
  CK_CUDA(chfsi::div_scalar_launch(static_cast<const double2*>(q0) + row0, nrm, V, nl, s));
  void* qfull = nullptr;
  if (gather_fn(user, V, nl, 1, &qfull) != 0 || !qfull) return fail(CHFSI_EINVAL, "gather failed");
  for (int i = 0; i < k; ++i) {
    const double2* q = V + (long long)i * nl;
    CK_CUDA(chfsi::gemv_rows_launch(hh, ldh, conj_h != 0, static_cast<const double2*>(qfull), u, n, done,
                                    s, nl));
    CK_CUDA(chfsi::dot_re_launch(q, u, nl, ctx->partial, al_d + i, done, s));
    CK(reduce(al_d + i, 1));
    CK_CUDA(chfsi::lanczos_residual_launch(u, q, i ? V + (long long)(i - 1) * nl : nullptr, al_d + i,
                                           i ? be_d + i - 1 : nullptr, r, nl, done, s));
    CK_CUDA(chfsi::colsdot_launch(V, nl, nl, i + 1, r, coef, done, s));
    CK(reduce(coef, 2LL * (i + 1)));
    CK_CUDA(chfsi::sub_vcoef_launch(V, nl, nl, i + 1, coef, r, done, s));
    CK_CUDA(chfsi::norm2sq_launch(r, nl, ctx->partial, nrm, done, s));
    CK(reduce(nrm, 1));
    CK_CUDA(chfsi::sqrt_scalar_launch(nrm, s));
    double2* qn = i + 1 < k ? V + (long long)(i + 1) * nl : nullptr;
    CK_CUDA(chfsi::lanczos_advance_launch(r, nrm, qn, be_d + i, st, i, k, nl, s));
    if (qn && (gather_fn(user, qn, nl, 1, &qfull) != 0 || !qfull))
      return fail(CHFSI_EINVAL, "gather failed");
  }
  chfsi::LanczosState hst;
  CK_CUDA(cudaMemcpyAsync(&hst, st, sizeof(hst), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaMemcpyAsync(alphas, al_d, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaMemcpyAsync(betas, be_d, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaStreamSynchronize(s));
  *steps = hst.steps;
  *beta_last = hst.beta_last;
  return CHFSI_OK;
}
