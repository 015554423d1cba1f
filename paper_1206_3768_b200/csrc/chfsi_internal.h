// Internal (C++) declarations shared by the kernel translation units and
// the C-ABI layer. Not part of the public interface (see include/chfsi.h).
#pragma once

#include <cuda_runtime.h>

namespace chfsi {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

// Counts launches of libchfsi's own kernels (chfsi_launch_count()).
void note_launch();

struct StepTiling {
  int bm;     // 0 = choose automatically; 32, 64 or 128 rows per CTA tile
  int bn;     // 16, 32 or 64 columns per CTA tile
  int split;  // grid override for tests/tuning (0 = all resident CTAs)
  int groups = 1;  // 1: one 8/16-warp tile group per CTA; 2: two 8-warp groups splitting k
  int product = 0; // complex product: 0 = process default, 3 = Gauss/3M, 4 = four real MMAs
  int warps = 0;   // warps per tile group: 0 = the registry's default for (bm, bn, groups)
};

// Stream-K scratch owned by the context: partial tiles + ready flags, and
// the CTA ticket counter at flags[max_grid] (logical CTA ids in dispatch order).
struct StepWorkspace {
  double* partials;
  unsigned* flags;    // [max_grid + 1]
  unsigned* epoch;    // host-side launch counter (flag generation)
  unsigned* tickets;  // host-side mirror of the device ticket counter
  int max_grid;
};

StepTiling choose_step_tiling(int n, int w);
// process-wide K1 complex-product default (3 or 4); returns the previous one, -1 if invalid
int set_complex_product(int product);
int complex_product();
// K1 3M k-slab depth in 128-byte halves (2 or 4); returns the previous, -1 if invalid
int set_k1_slab(int nh);
size_t step_workspace_doubles(int max_grid);
// CHFSI_K1_DEBUG & 8 diagnostics: copy the last K1 launch's per-CTA trace
// ([start, wait begin, wait end, end] globaltimer ns, smid) to host.
int step_trace_copy(unsigned long long* host, int max_ctas);
int step_grid_size(int bn, bool conj);

// K1: Ynext = alpha*(op(H) Ycur - c Ycur) - beta Yprev; Yprev may alias Ynext
// (or be null when beta == 0). op(H) = H (row-major read) or conj(H).
cudaError_t cheb_step_launch(const double2* h, long long ldh, bool conj_h, const double2* ycur,
                             long long ldc, const double2* yprev, long long ldp, double2* ynext,
                             long long ldn, int n, int w, double alpha, double c, double beta,
                             StepTiling tiling, const StepWorkspace& ws, cudaStream_t stream,
                             bool pdl = false);

// Row shard of K1 for the multi-GPU filter: compute `rows` output rows
// (H points at the shard's first row); Ycur may be in the rank-blocked
// layout (kblk rows per block, nblk blocks, block q = rows [q*kblk, ...)),
// and the epilogue's c*Ycur term then reads the shard's own rows at
// ycur_rows (ld ldcr).
struct RowShard {
  int rows;
  int kblk;   // 0: Ycur is plain column-major
  int nblk;
  const double2* ycur_rows;
  long long ldcr;
};
// peer_shift / npeer: fused all-gather — every output element is also stored
// at ynext + peer_shift[k] (elements), k < npeer <= 7 (peers' buffers mapped
// into this process; NVLink P2P stores from the epilogue).
cudaError_t cheb_step_rows_launch(const double2* h, long long ldh, bool conj_h, const double2* ycur,
                                  long long ldc, const double2* yprev, long long ldp, double2* ynext,
                                  long long ldn, int n, int w, double alpha, double c, double beta,
                                  const RowShard& shard, StepTiling tiling, const StepWorkspace& ws,
                                  cudaStream_t stream, const long long* peer_shift = nullptr,
                                  int npeer = 0, bool pdl = false);

// ---- auxiliary kernels (aux_kernels.cu) ----
// u = op(H) q for a row-major H (conj_h: conj(H)).
cudaError_t gemv_rows_launch(const double2* h, long long ldh, bool conj_h, const double2* q,
                             double2* u, int n, const int* done, cudaStream_t s, int rows = -1);
// ||x||^2 (no square root) and x <- sqrt(x) on one device scalar
cudaError_t norm2sq_launch(const double2* x, long long n, double* partial, double* out,
                           const int* done, cudaStream_t s);
cudaError_t sqrt_scalar_launch(double* x, cudaStream_t s);
// Deterministic reductions. partial buffers must hold kRedBlocks entries.
constexpr int kRedBlocks = 296;
constexpr int kRedThreads = 256;
// out = Re(x^H y) or ||x||_2 (op 0/1); x,y length n.
cudaError_t dot_re_launch(const double2* x, const double2* y, int n, double* partial, double* out,
                          const int* done, cudaStream_t s);
cudaError_t norm2_launch(const double2* x, long long n, double* partial, double* out,
                         const int* done, cudaStream_t s);
// dst = src and *out = ||src||_2 in one launch (counter: a zeroed device word the kernel re-arms)
cudaError_t copy_norm2_launch(const double2* src, double2* dst, long long n, double* partial,
                              unsigned* counter, double* out, cudaStream_t s);
// out[j] = x_j^H r for columns j < ncols of col-major V (ld).
cudaError_t colsdot_launch(const double2* v, long long ldv, int n, int ncols, const double2* r,
                           double2* out, const int* done, cudaStream_t s);
// r[i] -= sum_j V[i,j] coef[j]   (fixed j order)
cudaError_t sub_vcoef_launch(const double2* v, long long ldv, int n, int ncols,
                             const double2* coef, double2* r, const int* done, cudaStream_t s);

// Lanczos step pieces with device-side control state.
struct LanczosState {
  int done;
  int steps;
  double beta_last;
};
// whole k-step Lanczos in one cooperative kernel (lanczos.cu)
int lanczos_coop_grid(int n);
size_t lanczos_coop_workspace_bytes(int n, int k);
cudaError_t lanczos_coop_launch(const double2* h, long long ldh, bool conj_h, int n, int k,
                                const double2* q0, double2* V, void* ws, double* alphas,
                                double* betas, LanczosState* st, cudaStream_t s);
cudaError_t lanczos_residual_launch(const double2* u, const double2* q, const double2* qprev,
                                    const double* alpha_i, const double* beta_prev, double2* r,
                                    int n, const int* done, cudaStream_t s);
cudaError_t lanczos_advance_launch(const double2* r, const double* beta, double2* qnext,
                                   double* betas_i, LanczosState* st, int i, int k, int n,
                                   cudaStream_t s);

// res[j] = || HP[:,j] - lambda[j] P[:,j] ||_2  (col-major, one block per column)
// (squared: sums of squares, for row-sharded partial norms)
cudaError_t colnorm_residual_launch(const double2* hp, long long ldhp, const double2* p,
                                    long long ldp, const double* lambda, int n, int w,
                                    double* res, cudaStream_t s, bool squared = false);
// res[j] = || X[:,j] ||_2
cudaError_t colnorm_launch(const double2* x, long long ldx, int n, int w, double* res,
                           cudaStream_t s);
// A <- (A + A^H)/2 in place (square, col-major or row-major alike)
cudaError_t symmetrize_launch(double2* a, long long lda, int n, cudaStream_t s);
// out[0] = max |A - A^H|, out[1] = max |A|
cudaError_t herm_defect_launch(const double2* a, long long lda, int n, double* out,
                               cudaStream_t s);
// A <- conj(A) elementwise (m x n col-major block); also zero strict upper if tril
cudaError_t conj_inplace_launch(double2* a, long long lda, int m, int n, cudaStream_t s);
// dst = src^H (square, column-major, out of place)
cudaError_t conj_transpose_launch(const double2* src, long long lds, double2* dst, long long ldd, int n,
                                  cudaStream_t s);
cudaError_t zero_upper_launch(double2* a, long long lda, int n, cudaStream_t s);
// Q[:, j] *= conj(d_j / |d_j|), d_j = R[j, j] read from the (separate) diag array
cudaError_t phase_fix_launch(double2* q, long long ldq, int m, int n, const double2* rdiag,
                             cudaStream_t s);
// diag[j] = A[j, j]
cudaError_t extract_diag_launch(const double2* a, long long lda, int n, double2* diag,
                                cudaStream_t s);
// A[i,i] += coef * (*fro)^2  (shifted Cholesky-QR)
cudaError_t add_diag_shift_launch(double2* a, long long lda, int n, const double* fro, double coef,
                                  cudaStream_t s);
// acc[i] = (first ? 1 : acc[i]) * Re(R[i,i])
cudaError_t diag_accumulate_launch(const double2* r, long long ldr, int n, double* acc, bool first,
                                   cudaStream_t s);
// near-diagonal Hermitian eigensolver as one cooperative kernel (nd_persist.cu)
constexpr int kNdPersistMaxN = 256;
size_t nd_persist_ws_bytes(int n);
cudaError_t nd_persist_launch(const double2* a, long long lda, int n, double* w, double tol,
                              double bail, void* ws, double* status_dev, cudaStream_t s);
// near-diagonal Hermitian eigensolver pieces (nd_eig.cu)
cudaError_t nd_build_step_launch(const double2* g, long long ldg, int n, double2* x, long long ldx,
                                 double* stats, cudaStream_t s);
cudaError_t nd_ns_matrix_launch(double2* t, long long ldt, int n, double* defect, cudaStream_t s);
cudaError_t nd_sort_launch(const double2* g, long long ldg, int n, double* w, int* perm,
                           cudaStream_t s);
cudaError_t nd_gather_cols_launch(const double2* src, long long lds, int m, int n, const int* perm,
                                  double2* out, long long ldo, cudaStream_t s);
// y = x / *d (complex / real, round-to-nearest division)
cudaError_t div_scalar_launch(const double2* x, const double* d, double2* y, int n, cudaStream_t s);
// Y1 = alpha (HY - c Y0): the first filter step when H Y0 is already known
cudaError_t cheb_first_step_launch(const double2* hy, long long ldhy, const double2* y0, long long ldy,
                                   double2* out, long long ldo, int n, int w, double alpha, double c,
                                   cudaStream_t s);
// Linearised second Cholesky-QR pass: G = Q1^H Q1 = I + E -> M = I - tri(E)
// in place (upper; tri = strict upper + diag/2), out[0] = max|E_ij|,
// acc[i] *= 1 + E_ii/2, last[i] = 1 + E_ii/2 (the R2 diagonal to O(|E|^2)).
cudaError_t near_identity_update_launch(double2* g, long long ldg, int n, double* acc, double* last,
                                        double* out, cudaStream_t s);
// ---- Cholesky-QR2 panel kernels (panel_kernels.cu), widths <= kPanelMaxW ----
constexpr int kPanelMaxW = 192;
size_t panel_linv_bytes();
// after potrf (lower L in g): acc[i] = (first ? 1 : acc[i]) * L_ii, last[i] = L_ii
// (when given), the inverted 16x16 diagonal blocks of L into linv, *eps = 0
cudaError_t panel_post_potrf_launch(const double2* g, long long ldg, int n, double* acc, bool first,
                                    double* last, double2* linv, double* eps, cudaStream_t s);
// Y <- Y L^-H (m x n, ld; L lower n x n), one kernel, rows in shared memory
cudaError_t panel_trsm_lh_launch(double2* y, long long ld, int m, int n, const double2* l, long long ldl,
                                 const double2* linv, cudaStream_t s);
// linearised second pass in one kernel: Y <- Y (I - tri(G2 - I)) from the
// Gram matrix G2 (upper triangle read), *eps = max(*eps, max|E_ij|),
// acc[i] *= 1 + E_ii/2, last[i] = 1 + E_ii/2
cudaError_t panel_apply_near_identity_launch(double2* y, long long ld, int m, int n, const double2* g2,
                                             long long ldg, double* acc, double* last, double* eps,
                                             cudaStream_t s);
// Y[:, j] = X[:, j]
cudaError_t copy_cols_launch(const double2* x, long long ldx, double2* y, long long ldy, int m,
                             int n, cudaStream_t s);

}  // namespace chfsi
