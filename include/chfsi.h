/*
 * libchfsi — C-ABI of the B200-native ChFSI hot path (sm_100a).
 *
 * The reference (`spectral_chain`, pure Python + numpy/scipy) has no FFI:
 * its boundary is the Python functions re-exported by
 * `spectral_chain/__init__.py:15-80`. Each entry point below replaces the
 * numpy/LAPACK work behind one of those functions; the reference interface
 * it replaces is cited per function (paths relative to
 * /root/reference/pkg/src/spectral_chain/). INTEGRATION.md shows the ctypes
 * binding the reference would add.
 *
 * Conventions
 *  - Matrices are complex128 (interleaved re/im, 16 bytes), passed as plain
 *    `void*` DEVICE pointers owned by the caller, column-major with a
 *    leading dimension `ld*`, except the operator H of K1/K2 which is read
 *    row-major (`H[m*ldh + k]`); `conj_h = 1` reads conj(H), so a
 *    column-major Hermitian H can be passed unchanged.
 *  - Work is enqueued on the context's stream (chfsi_ctx_set_stream) and is
 *    stream-ordered; functions returning host values synchronise that stream.
 *  - Every reduction has a fixed order: results are bitwise reproducible
 *    run to run on the same device.
 *  - Return value: CHFSI_OK (0) or a negative CHFSI_E* code;
 *    chfsi_last_error() gives a thread-local message.
 */
#ifndef CHFSI_H_
#define CHFSI_H_

#if defined(__GNUC__)
#define CHFSI_API __attribute__((visibility("default")))
#else
#define CHFSI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CHFSI_OK 0
#define CHFSI_EINVAL -1     /* bad argument -> ValueError                        */
#define CHFSI_ECUDA -2      /* CUDA runtime failure                              */
#define CHFSI_ECUBLAS -3    /* cuBLAS failure                                    */
#define CHFSI_ECUSOLVER -4  /* cuSOLVER failure                                  */
#define CHFSI_ENOTPD -5     /* Cholesky pivot <= 0 -> NotPositiveDefiniteError    */
#define CHFSI_ERANK -6      /* rank-deficient panel -> RankDeficientError         */
#define CHFSI_EEIG -7       /* dense eigensolver failed -> EigenSolverError       */
#define CHFSI_ENCCL -8      /* NCCL failure                                      */

typedef struct chfsi_ctx chfsi_ctx;

CHFSI_API int chfsi_version(void);
CHFSI_API const char* chfsi_last_error(void);
/* Number of libchfsi kernel launches so far in this process (all devices). */
CHFSI_API long long chfsi_launch_count(void);

/* One context per device and host thread of use; owns cuBLAS/cuSOLVER
 * handles and a growable device workspace. */
CHFSI_API int chfsi_ctx_create(int device, chfsi_ctx** out);
CHFSI_API int chfsi_ctx_destroy(chfsi_ctx* ctx);
CHFSI_API int chfsi_ctx_set_stream(chfsi_ctx* ctx, void* cuda_stream);
/* Force the K1 tiling for tests and tuning: (bm, bn) = 64x16 | 64x32 |
 * 64x64 (8 warps, two CTAs per SM) or 128x16 | 128x32 (16 warps, one CTA per
 * SM), plus 32x32 | 32x64, grid = number of persistent CTAs (0 = all resident CTAs;
 * fewer CTAs exercise other stream-K splits). bm = 0 restores automatic. */
CHFSI_API int chfsi_ctx_set_tiling(chfsi_ctx* ctx, int bm, int bn, int grid);
/* With a forced tiling: groups = 2 selects the one-CTA-per-SM K1 whose two
 * 8-warp groups take alternate k-slabs of the same tile (64x16, 64x32). */
CHFSI_API int chfsi_ctx_set_step_groups(chfsi_ctx* ctx, int groups);
/* With a forced tiling: warps per tile group (4, 8 or 16; 0 = the default
 * variant of that tiling). A combination without a kernel fails at launch. */
CHFSI_API int chfsi_ctx_set_step_warps(chfsi_ctx* ctx, int warps);
/* Filter launch chains (default 2): with 2, chfsi_filter_z runs balanced
 * column halves as two concurrent launch chains (the context's stream and an
 * internal one, joined before returning) when the automatic tiling allows;
 * 1 = one chain (tests/tuning). */
CHFSI_API int chfsi_ctx_set_filter_chains(chfsi_ctx* ctx, int chains);

/* ---------------------------------------------------------------- K1 ---
 * One fused Chebyshev step (chfsi.py:203 / chfsi.py:206):
 *   Ynext = alpha*(op(H) Ycur - c Ycur) - beta Yprev
 * Yprev may alias Ynext (in-place ping-pong) or be NULL when beta == 0;
 * Ycur must not alias Ynext. alpha=1, c=0, beta=0 is the plain product H*Y
 * (the Rayleigh-Ritz H*panel of chfsi.py:342). */
CHFSI_API int chfsi_cheb_step_z(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                      const void* ycur, long long ldc, const void* yprev, long long ldp,
                      void* ynext, long long ldn, double alpha, double c, double beta);

/* Row shard of one Chebyshev step for the multi-GPU filter:
 * computes rows [r0, r0+rows) of Ynext = alpha*(H Ycur - c Ycur) - beta Yprev
 * where H_rows points at row r0 of H (row-major read, ld ldh, n columns).
 * Ycur is the FULL block, either column-major (kblk = 0, ld ldc) or in the
 * rank-blocked layout the NCCL all-gather produces (kblk rows per block,
 * nblk blocks; block q holds rows [q*kblk, (q+1)*kblk), column-major inside,
 * padding rows zero). ycur_rows / yprev / ynext address the shard's own rows
 * (ld ldcr / ldp / ldn); yprev may alias ynext. */
CHFSI_API int chfsi_cheb_step_rows_z(chfsi_ctx* ctx, int n, int rows, int w, const void* H_rows,
                                     long long ldh, int conj_h, const void* ycur, long long ldc,
                                     int kblk, int nblk, const void* ycur_rows, long long ldcr,
                                     const void* yprev, long long ldp, void* ynext, long long ldn,
                                     double alpha, double c, double beta);
/* Fused all-gather variant (multi-GPU over NVLink): additionally stores every
 * output element at the same position of npeer (<= 7) peer buffers,
 * peer_ynext[k] being the peer's equivalent of `ynext` mapped into this
 * process (CUDA IPC / symmetric memory). The all-gather then happens tile by
 * tile from K1's epilogue; the caller orders steps with a cross-rank
 * barrier. */
CHFSI_API int chfsi_cheb_step_rows_peers_z(chfsi_ctx* ctx, int n, int rows, int w, const void* H_rows,
                                           long long ldh, int conj_h, const void* ycur, long long ldc,
                                           int kblk, int nblk, const void* ycur_rows, long long ldcr,
                                           const void* yprev, long long ldp, void* ynext, long long ldn,
                                           double alpha, double c, double beta,
                                           const void* const* peer_ynext, int npeer);

/* Host-only: the filter's shift c and per-step (alpha_j, beta_j) exactly as
 * chebyshev_filter computes them (chfsi.py:198-207). alphas/betas hold deg. */
CHFSI_API int chfsi_filter_coeffs(int deg, double a, double b, double scale_ref, double* c,
                        double* alphas, double* betas);

/* Replaces chebyshev_filter(h, y, deg, window) (chfsi.py:179-208).
 * y0 is read only; the result lands in buf_a (deg odd) or buf_b (deg even)
 * and *result receives that pointer. y0 may equal buf_b (in place). */
CHFSI_API int chfsi_filter_z(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh, int conj_h,
                   const void* y0, long long ldy0, void* buf_a, void* buf_b, long long ldb,
                   int deg, double a, double b, double scale_ref, void** result);

/* Per-column degrees (SURVEY G4, config C5's adaptive filter): column j of
 * the result is the degree-degs[j] filter of Y0[:, j]; degs is a HOST array,
 * non-decreasing, each >= 1 (sort the columns first). One recurrence runs
 * for all columns and retires each as its degree is reached, so the work is
 * 8 n^2 sum(degs). Same buffers and aliasing rules as chfsi_filter_z. */
CHFSI_API int chfsi_filter_degrees_z(chfsi_ctx* ctx, int n, int w, const void* H, long long ldh,
                                     int conj_h, const void* y0, long long ldy0, void* buf_a,
                                     void* buf_b, long long ldb, const int* degs, double a, double b,
                                     double scale_ref, void** result);

/* Diagnostics: with CHFSI_K1_DEBUG=8 in the environment every K1 launch
 * records per-CTA [start, owner-wait begin, owner-wait end, end]
 * (%globaltimer ns) and the SM id; this copies the last launch's records
 * (5 values per CTA) and returns the number of CTAs (0: tracing off). */
CHFSI_API int chfsi_debug_k1_trace(unsigned long long* host, int max_ctas);

/* Introspection of the K1 tile choice for an (n, w) step. */
CHFSI_API int chfsi_step_tiling(int n, int w, int* bm, int* bn, int* split);

/* Complex-product formulation of K1 (process-wide; default 3 unless the
 * environment sets CHFSI_K1_PRODUCT=4): 3 = Gauss/3M, three real FP64 MMAs
 * per complex block (Cr = T1 - T2, Ci = T3 - T1 - T2), 4 = four real MMAs.
 * Both round like a complex GEMM to O(u) normwise; the 8-flop-per-complex-MAC
 * count of the metric is unchanged. Returns the previous setting (3 or 4),
 * or CHFSI_EINVAL; product = 0 only queries. */
CHFSI_API int chfsi_set_complex_product(int product);

/* K-slab depth of the 3M K1 kernels in 128-byte halves (process-wide):
 * 2 = 16 complex per TMA stage, 4 = 32 complex (default unless
 * CHFSI_K1_NH=2; half the stage barriers per MMA, same shared memory with half the
 * stages; tiles without a deep variant keep 16). Same arithmetic and
 * summation order either way. Returns the previous setting, or CHFSI_EINVAL;
 * halves = 0 only queries. No reference counterpart (tuning knob). */
CHFSI_API int chfsi_set_k1_slab(int halves);

/* Panel kernels of the Cholesky-QR2 orthonormalisation (process-wide; default
 * on unless CHFSI_PANEL_KERNELS=0): for panel widths <= 192 the triangular
 * solve Y L^-H and the linearised second pass run as one hand-written
 * row-parallel kernel each instead of cuBLAS ZTRSM / ZGEMM chains. on = 1 / 0
 * sets, -1 queries; returns the previous setting. Same algebra, results
 * agree to rounding. No reference counterpart (tuning knob; the reference's
 * QR is numpy's Householder, linalg.py:152-178). */
CHFSI_API int chfsi_set_panel_kernels(int on);

/* ---------------------------------------------------------------- K2 ---
 * k-step Lanczos with full reorthogonalization (chfsi.py:125-162): q0 is
 * the raw start vector (normalised on device), basis an n x k column-major
 * workspace (ld n). Writes alphas[0..steps), betas[0..steps-1), the final
 * residual norm and the step count to HOST memory. */
CHFSI_API int chfsi_lanczos_z(chfsi_ctx* ctx, int n, int k, const void* H, long long ldh, int conj_h,
                    const void* q0, void* basis, double* alphas, double* betas,
                    double* beta_last, int* steps);

/* Lanczos implementation (tests/tuning): 0 = one cooperative persistent
 * kernel for all k steps (default); 1 = one launch per operation. */
CHFSI_API int chfsi_ctx_set_lanczos_mode(chfsi_ctx* ctx, int mode);

/* ------------------------------------------------------- K3 / K4 (RR) ---
 * Plain ZGEMM C = alpha op(A) op(B) + beta C (cuBLAS; trans 'N','T','C'). */
CHFSI_API int chfsi_gemm_z(chfsi_ctx* ctx, char transa, char transb, int m, int n, int k, double alpha_re,
                 double alpha_im, const void* A, long long lda, const void* B, long long ldb,
                 double beta_re, double beta_im, void* C, long long ldc);

/* Two classical Gram-Schmidt passes of work against locked
 * (chfsi.py:251-253): work -= locked (locked^H work), twice. coef is an
 * nlocked x w scratch block (ld nlocked). */
CHFSI_API int chfsi_cgs_project_z(chfsi_ctx* ctx, int n, int nlocked, int w, const void* locked,
                        long long ldl, void* work, long long ldw, void* coef);

/* Householder QR orthonormalization with positive-real R diagonal
 * (linalg.py:152-178). Q overwrites Y. If any |R_ii| < 1e-13 ||Y||_F the
 * call returns CHFSI_ERANK, Y is left unmodified, and the offending column
 * indices (ascending) are written to dead[0..*ndead) (dead holds n ints). */
CHFSI_API int chfsi_qr_orthonormalize_z(chfsi_ctx* ctx, int m, int n, void* Y, long long ldy, int* dead,
                              int* ndead);

/* QR algorithm selection (tests/tuning): 0 (default) = Cholesky-QR2 (two
 * GEMM + potrf + TRSM passes), accepted when the second pass's R is the
 * identity to 1e-6, else shifted Cholesky-QR3 (three passes, Fukaya's shift),
 * else Householder — Householder also whenever a pivot fails or any
 * |R_ii| < 1e-11 ||Y||_F, so the reference's rank test is always decided by
 * Householder; 1 = Householder only; 2 = shifted Cholesky-QR3, then
 * Householder. All return the same (unique) Q with positive-real R diagonal. */
CHFSI_API int chfsi_ctx_set_qr_mode(chfsi_ctx* ctx, int mode);
/* Cholesky-QR2's second pass (default on): after the first pass
 * eps = max|Q1^H Q1 - I| ~ u cond(Y)^2; when eps <= 1e-8 the second factor is
 * taken to first order, R2 = I + tri(E) (strict upper + diag/2 of
 * E = Q1^H Q1 - I), and Q = Q1 (I - tri(E)) by one ZGEMM — the same
 * positive-diagonal QR to O(eps^2) without a second potrf + ZTRSM. eps > 1e-8
 * reruns the exact pass. on = 0 always runs the exact pass. */
CHFSI_API int chfsi_ctx_set_qr_linear2(chfsi_ctx* ctx, int on);

/* Dense Hermitian eigensolver (linalg.py:181-206): ascending values to the
 * DEVICE array w, eigenvectors overwrite A. */
CHFSI_API int chfsi_heevd_z(chfsi_ctx* ctx, int n, void* A, long long lda, double* w);

/* Rayleigh-Ritz eigensolver (chfsi.py:347): when G is near-diagonal (max
 * |G_ij| / |G_jj - G_ii| <= 0.25, the regime of every ChFSI loop after the
 * first few) it runs simultaneous first-order Jacobi steps (ZGEMM +
 * Newton-Schulz) until max|G_ij| <= tol * max(1, max|G_ii|) and sets
 * *used_fast = 1; otherwise, or if that fails, it is exactly chfsi_heevd_z.
 * tol <= 0 forces zheevd. Same outputs as chfsi_heevd_z. */
CHFSI_API int chfsi_heev_rr_z(chfsi_ctx* ctx, int n, void* A, long long lda, double* w, double tol,
                              int* used_fast);

/* res[j] = || HP[:,j] - lambda[j] P[:,j] ||_2 (chfsi.py:350); device arrays.
 * P and lambda may be NULL (plain column norms). */
CHFSI_API int chfsi_colnorm_residual_z(chfsi_ctx* ctx, int n, int w, const void* HP, long long ldhp,
                             const void* P, long long ldp, const double* lambda, double* res);
/* The squares ||HP[:,j] - lambda[j] P[:,j]||^2 (row-sharded partial sums). */
CHFSI_API int chfsi_colnorm_residual_sq_z(chfsi_ctx* ctx, int n, int w, const void* HP, long long ldhp,
                                          const void* P, long long ldp, const double* lambda,
                                          double* res);

/* ------------------------------------------------------------------ K5 ---
 * A <- (A + A^H)/2 in place (reduction.py:112, chfsi.py:346). */
CHFSI_API int chfsi_symmetrize_z(chfsi_ctx* ctx, int n, void* A, long long lda);
/* Hermitian validation (linalg.py:61-85): max|A - A^H| and max|A| to host. */
CHFSI_API int chfsi_herm_defect_z(chfsi_ctx* ctx, int n, const void* A, long long lda, double* defect,
                        double* maxabs);
/* A <- conj(A) for an m x n block (row-major <-> column-major of a Hermitian). */
CHFSI_API int chfsi_conj_z(chfsi_ctx* ctx, int m, int n, void* A, long long lda);
/* Lower Cholesky in place, strict upper zeroed (linalg.py:116-129).
 * Returns CHFSI_ENOTPD with *info = failing pivot (1-based). */
CHFSI_API int chfsi_potrf_z(chfsi_ctx* ctx, int n, void* A, long long lda, int* info);
/* B <- op(L)^-1 B (side 'L') or B op(L)^-1 (side 'R'), L lower non-unit
 * (linalg.py:132-149). trans 'N' or 'C'. */
CHFSI_API int chfsi_trsm_z(chfsi_ctx* ctx, char side, char trans, int m, int n, const void* L,
                 long long ldl, void* B, long long ldb);
/* to_standard (reduction.py:102-113): on entry A and B hold the pencil
 * (column-major, or row-major with rowmajor_in = 1); on exit B holds L
 * (lower, column-major) and A holds H = L^-1 A L^-H, re-symmetrised. */
CHFSI_API int chfsi_to_standard_z(chfsi_ctx* ctx, int n, void* A, long long lda, void* B, long long ldb,
                        int rowmajor_in, int* info);
/* Stream-ordered variants for pipelined sequences (no host synchronisation):
 * the potrf pivot status / (defect, max|A|) are copied to caller-owned
 * PAGE-LOCKED host memory and are valid once the stream has passed this
 * point; the caller raises the reference's exceptions then. */
CHFSI_API int chfsi_to_standard_async_z(chfsi_ctx* ctx, int n, void* A, long long lda, void* B,
                                        long long ldb, int rowmajor_in, int* info_host);
/* The same reduction with both triangular solves as block substitutions
 * whose off-diagonal products run on K1 (3M DMMA) and whose nb x nb diagonal
 * blocks use ZTRSM: Z = L^-1 A, then H = L^-1 Z^H (= Z L^-H). `work` is
 * caller-owned device memory for 2 n^2 complex (L^H and Z^H). */
CHFSI_API int chfsi_to_standard_k1_z(chfsi_ctx* ctx, int n, void* A, long long lda, void* B,
                                     long long ldb, int rowmajor_in, void* work, int* info_host);
CHFSI_API int chfsi_herm_defect_async_z(chfsi_ctx* ctx, int n, const void* A, long long lda,
                                        double* out_host);
/* back_transform (reduction.py:122-134): Y <- L^-H Y in place (backward block
 * substitution, off-diagonal products on K1). */
CHFSI_API int chfsi_back_transform_z(chfsi_ctx* ctx, int n, int nev, const void* L, long long ldl, void* Y,
                           long long ldy);

/* --------------------------------------------------------------- driver ---
 * The inner loop of chfsi_solve (chfsi.py:328-373) in native code: per pass
 * filter -> CGS against the locked block + QR with rank repair -> Rayleigh-
 * Ritz -> locking of leading converged Ritz pairs -> window refresh
 * (chfsi.py:264-271), until nev pairs are locked or max_repeats passes ran.
 * The caller sets up the start block (bufs[0], orthonormal), the window and
 * the workspace; the loop leaves its state and counters in the struct.
 * Optional host callbacks: `filter` replaces the single-GPU filter (the
 * row-sharded multi-GPU filter; `degs` is NULL or the sorted per-column
 * degrees), `fill` draws replacement columns for a rank-deficient panel (the
 * caller's RNG, reference draw order).
 * adaptive != 0: per-vector degrees capped at deg, from the
 * previous pass's Ritz values and residuals; the panel columns are reordered
 * by ascending degree before each filter (oracle/chfsi_oracle.py restates
 * the rule). */
typedef int (*chfsi_filter_cb)(void* user, const void* panel, void* other, long long ld, int width,
                               int deg, const int* degs, double a, double b, double scale_ref,
                               void** result);
typedef int (*chfsi_fill_cb)(void* user, void* block, long long ld, int rows, const int* cols,
                             int ncols);
/* Row-sharded (multi-GPU) loop: in-place sum over the ranks of `count`
 * doubles at the device pointer `buf`, complete on return (stream-ordered
 * after the context's stream); identical result on every rank. */
typedef int (*chfsi_allreduce_cb)(void* user, void* buf, long long count);
/* out_local = rows row0..row0+n_local of H * P, from this rank's rows of P
 * (ld n_local); complete or stream-ordered on return. */
typedef int (*chfsi_hp_cb)(void* user, const void* panel_local, void* out_local, long long ld,
                           int width);
/* *full (n x width, ld n, owned by the caller of the loop) = all ranks' rows
 * of the local block (ld ld_local). */
typedef int (*chfsi_gather_cb)(void* user, const void* local, long long ld_local, int width,
                               void** full);

typedef struct chfsi_loop {
  /* problem and device workspace (in) */
  int n, blk, nev, deg, max_repeats;
  int adaptive, deg_min;     /* per-vector adaptive degree (deg = cap) */
  double tol;
  double rr_fast_tol;        /* > 0: near-diagonal RR eigensolver tried first (else zheevd only) */
  const void* H;
  long long ldh;
  int conj_h;
  void* bufs[2];             /* n x blk panels, ld n; bufs[0] holds the orthonormal start block */
  void* hp;                  /* n x blk */
  void* hp_rot;              /* n x blk */
  void* locked;              /* n x nev, ld n */
  void* g;                   /* blk x blk, ld blk */
  void* coef;                /* nev x blk, ld nev */
  double* ritz_d;            /* device, blk */
  double* res_d;             /* device, blk */
  int* perm_d;               /* device, blk ints (adaptive column order); may be NULL otherwise */
  void* tail;                /* NULL, or n x blk (ld n): filled at exit with [locked | unlocked
                                remainder of the final panel], the chained warm start */
  /* Row-sharded mode (multi-GPU): every n x w block above holds
   * only rows row0 .. row0+n_local-1 of this rank (ld n_local, so `n` stays
   * the global dimension); n x w products run on local rows and their w x w
   * / w-sized results are summed with `allreduce`; H*P comes from `hp` and
   * the filter from `filter`; the rare full-matrix fallbacks (Householder,
   * rank repair) use `gather`. allreduce == NULL: single GPU (n_local = n). */
  int row0, n_local;
  chfsi_allreduce_cb allreduce;
  chfsi_hp_cb hp_fn;
  chfsi_gather_cb gather;
  chfsi_filter_cb filter;    /* NULL: chfsi_filter_z on this context */
  chfsi_fill_cb fill;        /* NULL: rank deficiency is an error */
  void* user;
  /* window and loop state (in/out) */
  double win_a, win_b, win_scale_ref;
  int inner_loops, nlocked, pb, off, width, converged;
  int last_rot_pb, last_width, last_nlock; /* the final pass's rotated panel */
  /* host outputs (caller-owned arrays) */
  double* locked_vals;       /* nev, in locking order */
  double* locked_res;        /* nev */
  int* locked_per_loop;      /* max_repeats */
  double* ritz;              /* blk: the final pass's Ritz values */
  double* res;               /* blk: and residual norms */
  int* degs;                 /* blk: the next pass's sorted per-column degrees (adaptive) */
  /* counters (SolveReport, chfsi.py:101-122) and device phase times */
  long long filtered_vectors, matvecs, residual_check_matvecs, filter_launches, rr_fast_eigs;
  long long filter_degree_sum;  /* sum over passes and columns of the filter degree */
  double filter_flops;
  double t_filter, t_ortho, t_rr; /* seconds */
  /* in: 1 = from the second pass on, the filter's first step reuses H*P of the
   * previous Rayleigh-Ritz (rotated, unlocked columns == H * the next panel
   * to rounding), so it is elementwise instead of a K1 product (single GPU,
   * fixed degree; ignored with `filter`, `allreduce` or `adaptive`) */
  int reuse_hp;
  /* out: K1 launches / FLOPs the filter actually executed (filter_launches
   * and filter_flops stay the algorithmic deg-per-pass counts) */
  long long filter_k1_launches;
  double filter_k1_flops;
  /* out: passes whose speculative Cholesky-QR2 (acceptance test judged at
   * the pass's readback, no host round trip inside the QR) was rejected and
   * redone on the full QR path, together with their Rayleigh-Ritz */
  long long qr_redone;
} chfsi_loop;

CHFSI_API int chfsi_solve_loop_z(chfsi_ctx* ctx, chfsi_loop* loop);

/* Row-sharded Lanczos bound (multi-GPU, chfsi.py:125-162): this rank holds
 * rows row0 .. row0+n_local-1 of H (H_rows, row-major rows, conj_h as for
 * K1) and of the n x k basis (V_local, ld n_local); q0 is the full start
 * vector (replicated). Per step: GEMV on local rows against the gathered
 * vector, partial alpha / reorthogonalisation / norm sums completed by
 * `allreduce` (in place, stream-ordered), the next vector gathered with
 * `gather` (width 1). ws: chfsi_lanczos_rows_ws_bytes(n_local, k) device
 * bytes owned by the caller (the allreduce callback receives pointers into
 * it). Outputs as chfsi_lanczos_z, identical on every rank. */
CHFSI_API long long chfsi_lanczos_rows_ws_bytes(int n_local, int k);
CHFSI_API int chfsi_lanczos_rows_z(chfsi_ctx* ctx, int n, int k, const void* H_rows, long long ldh,
                                   int conj_h, int row0, int n_local, const void* q0, void* V_local,
                                   void* ws, chfsi_allreduce_cb allreduce, chfsi_gather_cb gather,
                                   void* user, double* alphas, double* betas, double* beta_last,
                                   int* steps);

#ifdef __cplusplus
}
#endif

#endif /* CHFSI_H_ */
