// Private to libchfsi's C-ABI translation units (chfsi_abi.cu,
// chfsi_loop.cu): the context object and the status-returning check macros.
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <string>

#include "../../include/chfsi.h"
#include "chfsi_internal.h"

struct chfsi_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  void* ws = nullptr;  // cuSOLVER workspace (grown on demand)
  size_t ws_bytes = 0;
  void* scratch = nullptr;  // n-sized vectors (grown on demand)
  void* eig_ws = nullptr;   // near-diagonal eigensolver work (grown on demand)
  size_t eig_ws_bytes = 0;
  size_t scratch_bytes = 0;
  double* partial = nullptr;  // kRedBlocks doubles
  double* scalars = nullptr;  // 16 doubles
  int* dinfo = nullptr;
  chfsi::LanczosState* lstate = nullptr;
  chfsi::StepTiling tiling{0, 0, 0};  // K1 tile override (bm == 0: automatic)
  chfsi::StepWorkspace step_ws{nullptr, nullptr, nullptr, 0};
  int qr_mode = 0;  // 0: shifted Cholesky-QR3 with Householder fallback; 1: Householder
  bool qr_linear2 = true;  // Cholesky-QR2: linearised second pass when |Q1^H Q1 - I| <= 1e-8
  int lanczos_mode = 0;  // 0: cooperative single kernel; 1: one launch per operation
  unsigned step_epoch = 0;
  unsigned step_tickets = 0;
  cudaEvent_t loop_ev[8] = {};  // chfsi_solve_loop_z phase timers (two sets, alternating passes)
  // second filter stream (two column halves of the filter run concurrently,
  // one CTA per SM each) with its own stream-K scratch
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  chfsi::StepWorkspace step_ws2{nullptr, nullptr, nullptr, 0};
  unsigned step_epoch2 = 0;
  unsigned step_tickets2 = 0;
  int filter_chains = 2;  // 1: one launch chain per filter (chfsi_ctx_set_filter_chains)
  void* pinned = nullptr;  // page-locked host staging for small readbacks (grown on demand)
  size_t pinned_bytes = 0;
  // deferred Cholesky-QR acceptance test (native loop): the checks' inputs
  // land here and are judged after the pass's own synchronisation
  void* qr_pinned = nullptr;
  size_t qr_pinned_bytes = 0;
  bool qr_pending = false;
  int qr_pending_n = 0;
  double* nd_pinned = nullptr;  // page-locked status of the speculative near-diagonal eigensolver
  bool nd_pending = false;
  unsigned* red_counter = nullptr;  // ticket word of the single-launch reductions (zero between launches)
  double2* panel_linv = nullptr;  // inverted diagonal blocks of the Cholesky-QR factor (panel_kernels.cu)
};

namespace chfsi {
// Page-locked host buffer of at least `bytes` owned by the context (for the
// small device->host readbacks that drive host decisions).
int ensure_pinned(chfsi_ctx* ctx, size_t bytes);
// Cholesky-QR2 with its acceptance test deferred: the panel is backed up,
// orthonormalised (CholQR2, linearised second pass) and the test's inputs
// queued to page-locked memory WITHOUT a host synchronisation; after the
// caller's next stream synchronisation `qr_deferred_verdict` judges them
// exactly as chfsi_qr_orthonormalize_z would. On rejection
// `qr_deferred_restore` puts the panel back as it was before the QR.
int qr_orthonormalize_deferred(chfsi_ctx* ctx, int m, int n, void* Y, long long ldy);
int qr_deferred_verdict(chfsi_ctx* ctx, bool* accept);
int qr_deferred_restore(chfsi_ctx* ctx, int m, int n, void* Y);
// Speculative Rayleigh-Ritz eigensolver (native loop): the cooperative
// near-diagonal solver is queued WITHOUT waiting for its verdict — the
// caller goes on queuing the rotations and residual norms as if it had
// succeeded and judges it (`heev_rr_verdict`) after the pass's own
// synchronisation. On failure A is untouched (the solver's contract) and
// the caller redoes the step with zheevd. *queued = false when the solver
// does not apply (width, tolerance, CHFSI_ND_PERSIST=0): nothing was done.
int heev_rr_speculative(chfsi_ctx* ctx, int n, void* A, long long lda, double* w, double tol, bool* queued);
int heev_rr_verdict(chfsi_ctx* ctx, bool* done);
// chfsi_filter_z with an optional known first product hy0 = H y0 (ld ldhy0):
// the first recurrence step is then elementwise (the native loop passes the
// previous Rayleigh-Ritz's rotated H P)
int filter_z_impl(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                  const void* y0, long long ldy0, const void* hy0, long long ldhy0, void* buf_a,
                  void* buf_b, long long ldb, int deg, double a, double b, double scale_ref,
                  void** result);
// chfsi_filter_degrees_z with the same optional known first product
int filter_degrees_impl(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                        const void* y0, long long ldy0, const void* hy0, long long ldhy0,
                        void* buf_a, void* buf_b, long long ldb, const int* degs, double a, double b,
                        double scale_ref, void** result);
// Records `msg` as this thread's chfsi_last_error() and returns `code`.
int fail(int code, const std::string& msg);
}  // namespace chfsi

#define CK_CUDA(expr)                                                                \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return chfsi::fail(CHFSI_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
  } while (0)
#define CK_BLAS(expr)                                                                        \
  do {                                                                                       \
    cublasStatus_t _s = (expr);                                                              \
    if (_s != CUBLAS_STATUS_SUCCESS)                                                         \
      return chfsi::fail(CHFSI_ECUBLAS, std::string(#expr) + ": cublas status " + std::to_string(_s)); \
  } while (0)
#define CK_SOLVER(expr)                                                                     \
  do {                                                                                      \
    cusolverStatus_t _s = (expr);                                                           \
    if (_s != CUSOLVER_STATUS_SUCCESS)                                                      \
      return chfsi::fail(CHFSI_ECUSOLVER,                                                          \
                  std::string(#expr) + ": cusolver status " + std::to_string(_s));          \
  } while (0)
#define CK_ARG(cond, msg) \
  do {                    \
    if (!(cond)) return chfsi::fail(CHFSI_EINVAL, msg); \
  } while (0)
#define CK(expr)              \
  do {                        \
    int _r = (expr);          \
    if (_r != CHFSI_OK) return _r; \
  } while (0)

