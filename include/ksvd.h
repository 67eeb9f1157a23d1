/*
 * ksvd.h -- C ABI of the B200-native Golub-Kahan (GK) bidiagonalization path.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `krysvd` (arXiv 2104.10785).  The reference is pure Python/numpy; it
 * has no FFI of its own.  Its plug-in surface for this path is the
 * `LinearOperator` protocol and the three entry points built on it:
 *
 *   reference                                         replaced by
 *   ------------------------------------------------  -----------------------------
 *   linops.py:160-161  MatrixOperator.matvec  A @ x   ksvd_matvec
 *   linops.py:163-164  MatrixOperator.rmatvec A.T @ y ksvd_rmatvec
 *   linops.py:166-167  MatrixOperator.matmat  A @ X   ksvd_matmat
 *   linops.py:82-86    _check_matrix (coerce to f64)  ksvd_matrix_from_host
 *   bidiag.py:111-184  bidiagonalize (the GK loop)    ksvd_gk_run + ksvd_run_info
 *   bidiag.py:95-108   _terminal_column               ksvd_run_extend
 *   bidiag.py:180-184  BidiagState.Q / .P (copies)    ksvd_run_bases
 *   fsvd.py:63-134     symtridiag_eig                 ksvd_symtridiag_eig (host)
 *   fsvd.py:191-201    V=P@G, U=A V/sigma, CGS2 cut,  ksvd_ritz
 *                      fix_signs (linops.py:271-282)
 *
 * The Python host driver (paper_2104_10785_b200/) binds these through
 * ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Every function returns an int status: KSVD_OK (0), KSVD_ERUNTIME (1,
 *    CUDA/NCCL failure -> RuntimeError), KSVD_ECONFIG (2 -> ConfigError,
 *    CLI exit 2 in the reference cli.py:369-374), KSVD_ENUMERIC (3 ->
 *    NumericalError, CLI exit 3).  ksvd_last_error() returns the
 *    thread-local message of the last failure.
 *  - Host buffers are caller-owned, contiguous, read/written only during
 *    the call.  Calls are synchronous on return.
 *  - Vectors and scalars are always double.  dtype selects only the
 *    storage of A (KSVD_F64, or KSVD_F32 whose entries are exact in f64,
 *    so products equal the reference run on the up-cast matrix up to
 *    summation order).
 *  - Multi-GPU: one process per GPU.  A is row-sharded: each rank holds
 *    rows [row0, row0 + m_local).  Left vectors (q, Q, U) are row-sharded,
 *    right vectors (p, P, V) are replicated.  Host vectors passed for the
 *    left side are LOCAL rows; right-side vectors are full length n.
 *  - Matrices stored column-major in host buffers below are "cols x rows"
 *    contiguous, i.e. column j starts at buf + j*rows.
 */
#ifndef KSVD_H
#define KSVD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KSVD_OK 0
#define KSVD_ERUNTIME 1
#define KSVD_ECONFIG 2
#define KSVD_ENUMERIC 3

#define KSVD_F64 0
#define KSVD_F32 1

/* ksvd_run_info flags */
#define KSVD_RUN_EARLY 1       /* terminated_early (bidiag.py:159,175)        */
#define KSVD_RUN_DEGENERATE 2  /* alpha_1 < eps     (bidiag.py:142-145)        */
#define KSVD_RUN_BETA_BREAK 4  /* beta_{k'+1} < eps (bidiag.py:158-164): the   */
                               /* caller completes Q with ksvd_run_extend      */
#define KSVD_RUN_ALPHA_BREAK 8 /* alpha_{k'+1} < eps (bidiag.py:174-176)       */

#define KSVD_NCCL_UID_BYTES 128
#define KSVD_PX_HANDLE_BYTES 64

typedef struct ksvd_ctx ksvd_ctx;
typedef struct ksvd_mat ksvd_mat;
typedef struct ksvd_run ksvd_run;

/* ---- library / context ------------------------------------------------ */
const char *ksvd_last_error(void);
int ksvd_version(void);
int ksvd_device_count(int *count);
/* Fill `uid` (KSVD_NCCL_UID_BYTES) with a fresh ncclUniqueId (rank 0). */
int ksvd_nccl_unique_id(char *uid);
/* nranks == 1: uid may be NULL and no communicator is created. */
int ksvd_ctx_create(int device, int rank, int nranks, const char *uid,
                    ksvd_ctx **out);
int ksvd_ctx_destroy(ksvd_ctx *ctx);
int ksvd_ctx_sync(ksvd_ctx *ctx);
/* Synchronise and return the device's freed stream-ordered pool memory to
 * the system (matrices and runs are pool allocations, kept mapped between
 * calls so the GK loop never unmaps; after freeing a large matrix this
 * makes the memory available to other allocators). */
int ksvd_ctx_release_pool(ksvd_ctx *ctx);
/* Per-kernel-class device timing (CUDA events on the launching stream). */
int ksvd_ctx_set_profiling(ksvd_ctx *ctx, int on);
/* cls: 0 gemv_n (A p), 1 gemv_t (A^T q), 2 CGS2 + norms, 3 other,
 * 4 product finalisation (split sums, axpy), 5 whole-loop resident kernel
 * (small matrices); returns launches and ms */
int ksvd_ctx_kernel_stats(ksvd_ctx *ctx, int cls, int64_t *launches,
                          double *ms);
int ksvd_ctx_reset_stats(ksvd_ctx *ctx);
/* Total kernel launches issued by this context since the last reset. */
int ksvd_ctx_launch_count(ksvd_ctx *ctx, int64_t *launches);
/* Device time (ms) between two context-stream marks; used by bench. */
int ksvd_ctx_mark(ksvd_ctx *ctx, int slot);
int ksvd_ctx_elapsed(ksvd_ctx *ctx, int slot0, int slot1, float *ms);
/* NVLink peer exchange (multi-rank; replaces ncclAllReduce for the GK
 * step's vectors up to `slot` doubles, reference counterpart: none -- the
 * reference is single-process).  Collective, in two halves around the
 * host-side all-gather of the handles: ksvd_px_export allocates this
 * rank's receive area and writes its CUDA IPC handle (KSVD_PX_HANDLE_BYTES);
 * ksvd_px_open maps every peer's area (handles: nranks x 64 bytes in rank
 * order), self-tests against NCCL and enables the exchange only if every
 * rank agrees (ksvd_px_enabled reports the outcome). */
int ksvd_px_export(ksvd_ctx *ctx, int64_t slot, unsigned char *handle);
int ksvd_px_open(ksvd_ctx *ctx, const unsigned char *handles);
int ksvd_px_enabled(ksvd_ctx *ctx, int *on);

/* ---- matrices ----------------------------------------------------------
 * rows: host pointer to the m_local local rows (row-major, src_ld elements
 * between rows) of the global m x n matrix; row0 = first global row.
 * Device layout: row-major, leading dimension padded to a 16-byte multiple
 * (KSVD_LDA_BYTES overrides), padding 0. */
int ksvd_matrix_from_host(ksvd_ctx *ctx, const void *rows, int64_t m_global,
                          int64_t n, int64_t row0, int64_t m_local,
                          int64_t src_ld, int dtype, ksvd_mat **out);
/* Same, from a device pointer (e.g. a torch tensor), copied into layout. */
int ksvd_matrix_from_device(ksvd_ctx *ctx, const void *rows, int64_t m_global,
                            int64_t n, int64_t row0, int64_t m_local,
                            int64_t src_ld, int dtype, ksvd_mat **out);
int ksvd_matrix_free(ksvd_mat *mat);
int ksvd_matrix_shape(ksvd_mat *mat, int64_t *m_global, int64_t *n,
                      int64_t *row0, int64_t *m_local, int *dtype,
                      int64_t *ld);
/* Copy local rows back (row-major, n per row). */
int ksvd_matrix_to_host(ksvd_mat *mat, void *rows);

/* y_local = A_local x            (x: n, y: m_local)          linops.py:161 */
int ksvd_matvec(ksvd_mat *mat, const double *x, double *y);
/* z = sum_ranks A_local^T y_local (y: m_local, z: n)         linops.py:164 */
int ksvd_rmatvec(ksvd_mat *mat, const double *y, double *z);
/* Y_local = A_local X (X: n x k column-major, Y: m_local x k col-major)  */
int ksvd_matmat(ksvd_mat *mat, const double *X, int k, double *Y);

/* ---- the GK loop -------------------------------------------------------
 * q1_local: the LOCAL rows of the normalized start vector q_1 (generated
 * by the caller from the reference's substream(seed, GK_START) so the
 * first column is bit-identical, bidiag.py:126-131).  Runs until k_max
 * steps or breakdown (bidiag.py:151-178).  The bases stay on the device. */
int ksvd_gk_run(ksvd_mat *mat, int k_max, double eps, int reorth_passes,
                const double *q1_local, ksvd_run **out);
/* alphas: capacity k_max, betas: capacity k_max+1 (betas[0] is filled
 * by the caller; the library writes alphas[0..k'-1] and betas[1..k'], i.e.
 * beta_{k'+1} included -- the sub-threshold value on a beta breakdown).  On
 * an alpha breakdown (k' < k_max) alphas[k'] receives the sub-threshold
 * alpha_{k'+1}, which the reference drops (bidiag.py:174-176); callers
 * that mirror the reference read alphas[0..k'-1] only. */
int ksvd_run_info(ksvd_run *run, int *k_prime, int *flags, double *alphas,
                  double *betas);
/* Terminal column (bidiag.py:95-108), one attempt: v = (v_local or the
 * stored residual w when v_local == NULL) / nrm, CGS2 against Q[:, :k'],
 * accepted iff ||v|| > 0.5, in which case Q[:, k'] = v/||v||. */
int ksvd_run_extend(ksvd_run *run, const double *v_local, double nrm,
                    int *accepted);
/* Q: q_cols columns of m_local rows; P: p_cols columns of n rows.  NULL
 * skips a side. */
int ksvd_run_bases(ksvd_run *run, double *Q, int q_cols, double *P,
                   int p_cols);
/* Ritz assembly (fsvd.py:191-201): V = P[:, :k'] G (G: k' x take col-major)
 * U = A V / sigma, optional CGS2 column filter with cut at 1e-2
 * (fsvd.py:142-155), sign fix (linops.py:271-282).  U: m_local x take,
 * V: n x take (column-major); n_good receives the kept column count. */
int ksvd_ritz(ksvd_run *run, const double *G, const double *sigma, int take,
              int orthonormalize_u, double *U, double *V, int *n_good);
/* ---- restarted mode (beyond reference semantics) ---
 * Thick restart of a finished, non-broken-down run of k = k' steps, in the
 * transposed ("A^T Q = P T") form where T is the k x k upper bidiagonal of
 * alphas (diagonal) and betas (superdiagonal): with T = Uh diag(s) Vh^T,
 * keep l Ritz pairs -- Q[:, :l] = Q[:, :k] X, Q[:, l] = q_{k+1},
 * P[:, :l] = P[:, :k] Y (X = Vh[:, :l], Y = Uh[:, :l], both k x l
 * column-major) -- then z = A^T q_{l+1}, CGS2 against P[:, :l] (the
 * coefficients are the restart spike rho_i = beta_{k+1} Uh[k-1, i]),
 * alpha_{l+1} = ||z||, and resume the standard loop at step l+1 up to
 * k_new.  ksvd_run_info then reports the new alphas[l..k'-1] and
 * betas[l+1..k'] (entries below are zero). */
int ksvd_run_restart(ksvd_run *run, int l, const double *X, const double *Y, int k_new);
/* U = Q[:, :kq] X (m_local x take), V = P[:, :kp] Y (n x take), sign fix
 * (linops.py:271-282 rule on V).  X: kq x take, Y: kp x take col-major. */
int ksvd_run_ritz_bases(ksvd_run *run, const double *X, int kq, const double *Y, int kp,
                        int take, double *U, double *V);
int ksvd_run_free(ksvd_run *run);

/* ---- synthetic matrices (BASELINE.json configs 3-5) -----------------------
 * A = P diag(s) Q^T + noise * G generated in HBM (no host copy): P (m x r),
 * Q (n x r) orthonormal (CholeskyQR2 of counter-based Gaussians), G iid
 * N(0,1) from Philox4x32-10 keyed by (seed, global index).  Entry arithmetic
 * is fixed by include/ksvd_gen.h so the host oracle regenerates the same
 * rows from the factors (ksvd_matrix_gen_factors).  Each rank generates its
 * row shard [row0, row0 + m_local) with row0 / m_local given by the
 * balanced contiguous partition (linops.row_partition). */
#define KSVD_SPEC_HARMONIC 0 /* s_i = s0 / i                         */
#define KSVD_SPEC_EXP 1      /* s_i = s0 * exp(-i / p)               */
#define KSVD_SPEC_GEOM 2     /* s_i = s0 * 10^(-p (i-1) / (r-1))     */
typedef struct ksvd_gen_spec {
  int64_t m, n;
  int32_t rank;
  int32_t dtype; /* KSVD_F64 / KSVD_F32 storage */
  uint64_t seed;
  int32_t spectrum;
  int32_t pad;
  double s0, p;
  double noise;
} ksvd_gen_spec;
int ksvd_matrix_generate(ksvd_ctx *ctx, const ksvd_gen_spec *spec, ksvd_mat **out);
/* Ps_local = P diag(s) for the local rows (m_local x r row-major), Q (n x r
 * row-major); r receives the rank.  Either pointer may be NULL. */
int ksvd_matrix_gen_factors(ksvd_mat *mat, double *Ps_local, double *Q, int *r);

/* ---- factored operator L C R^T (reference linops.py:176-205) -----------
 * FactoredOperator(left d1 x s1, core s1 x s2, right d2 x s2): every
 * product costs O((d1 + d2) s) and nothing of size d1 x d2 is formed.
 * left_rows = this rank's rows [row0, row0 + mloc) of `left` (row-major, s1
 * per row); core and right are full (row-major).  The handle is a ksvd_mat
 * usable with every product / GK / Ritz entry point; ksvd_matrix_to_host
 * and ksvd_matrix_to_klrm return KSVD_ECONFIG (no dense rows). */
int ksvd_matrix_from_factors(ksvd_ctx *ctx, const double *left_rows, const double *core,
                             const double *right, int64_t m, int64_t n, int64_t s1,
                             int64_t s2, int64_t row0, int64_t mloc, ksvd_mat **out);

/* ---- KLRM snapshots (reference matrixio.py:15-46) ------------------------
 * Little-endian header "<4sIQQ" (magic KLRM, u32 version 1, u64 rows, u64
 * cols) + rows*cols f64 row-major payload.  The reader streams this rank's
 * row shard straight into HBM through two pinned chunk buffers (file reads
 * overlap the host-to-device copies; the payload never exists whole in host
 * memory); dtype selects the device storage (KSVD_F32 rounds on the device).
 * The writer streams the local rows back at their file offsets (rank 0 also
 * writes the header), so N ranks write one file.  Format errors ->
 * KSVD_ECONFIG with the reference's messages. */
int ksvd_matrix_from_klrm(ksvd_ctx *ctx, const char *path, int dtype, ksvd_mat **out);
int ksvd_matrix_to_klrm(ksvd_mat *mat, const char *path);

/* ---- host spectral stage ------------------------------------------------
 * All eigenpairs of the symmetric tridiagonal (d, e), descending
 * (fsvd.py:63-134, implicit-shift QL, deflation |e| <= eps(|d_m|+|d_m+1|),
 * 64 sweeps max).  G: n x n column-major or NULL when vectors == 0. */
int ksvd_symtridiag_eig(int n, const double *d, const double *e, int vectors,
                        double *theta, double *G);
/* theta (descending) = squared singular values of the (k+1) x k lower
 * bidiagonal B (alphas[0..k-1], betas[1..k]) = eigenvalues of B^T B, each to
 * high relative accuracy (bisection on the Golub-Kahan tridiagonal); the
 * rank estimator's "tiny bidiagonal SVD" (rank.py:64). */
int ksvd_bidiag_sv2(int k, const double *alphas, const double *betas, double *theta);
/* Dense SVD T = U diag(s) V^T of a small k x k matrix (column-major; s
 * descending): the projected matrix of the restarted mode, whose first
 * rows carry the restart spike and so is not bidiagonal (one-sided Jacobi,
 * high relative accuracy).  No reference counterpart: SURVEY.md 8(f) row 3
 * (Ritz-vector restarts are a non-goal of the reference). */
int ksvd_dense_svd(int k, const double *T, double *U, double *s, double *V);
/* The same SVD in one CTA on the device (parallel round-robin Jacobi, the
 * north star's "single-CTA kernel" option); falls back to the host routine
 * when 2 k^2 doubles exceed the CTA's shared memory. */
int ksvd_dense_svd_dev(ksvd_ctx *ctx, int k, const double *T, double *U, double *s,
                       double *V);

#ifdef __cplusplus
}
#endif
#endif /* KSVD_H */
