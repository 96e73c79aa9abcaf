/*
 * trplk.h -- C ABI of the B200-native TRPL+K hot path (libtrplk.so).
 *
 * TRPL+K is the thick-restart preconditioned Lanczos method with +K (locally
 * optimal) restarting of arXiv 1711.10128 for the p algebraically smallest
 * eigenpairs of a sparse symmetric pencil A v = lambda B v with B SPD
 * (eq 1.1).  One call to trplk_solve runs Algorithm 1
 * (alg:trpl+k) entirely on the GPU: the projected inner
 * Lanczos step of eq 3.1 with the Jacobi preconditioner,
 * CGS2 reorthogonalisation in the B-inner product, the +K augmentation
 * (Alg. 1 steps 6-8), the Rayleigh-Ritz eigensolve of T
 * (step 11), the basis rotation U*Y (steps 11/15) and the soft-locking
 * residual test (steps 12-14).  The readings of ambiguous passages are the
 * R1-R20 of DESIGN.md.
 *
 * Conventions
 *  - All floating point is IEEE fp64.  Integers in CSR inputs are int64.
 *  - Matrices are CSR (0-based), both triangles stored, column ids strictly
 *    increasing within a row.  A rank passes only ITS rows [row_begin,row_end)
 *    (row pointers local, column ids global).
 *  - Every call returns a trplk_status; no exception crosses the ABI.  On a
 *    non-OK status trplk_last_error(ctx) gives a one-line reason.
 *  - A context is single-solve-at-a-time and not thread-safe; it may be reused
 *    for several solves.
 *  - Ownership: input CSR arrays stay owned by the caller (copied at create;
 *    may be freed afterwards).  All device memory is obtained through the
 *    optional trplk_allocator (else cudaMalloc) and released by trplk_destroy.
 *    Output buffers are caller-allocated.
 *  - `stream` is a cudaStream_t (passed as void*, the caller's stream; all
 *    work of the context is ordered on it).
 */
#ifndef TRPLK_H
#define TRPLK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TRPLK_ABI_VERSION 2
#define TRPLK_MAX_BASIS 64 /* largest max_basis (q) supported by the device kernels */

typedef enum {
    TRPLK_OK = 0,
    TRPLK_EINVAL = 1,        /* bad argument (see trplk_last_error) */
    TRPLK_NOT_CONVERGED = 2, /* max_cycles reached; outputs hold the current best (R19) */
    TRPLK_BREAKDOWN = 3,     /* basis exhausted (seed + 3 random replacements dependent); outputs filled */
    TRPLK_ECUDA = 4,         /* CUDA error; outputs undefined */
    TRPLK_ENCCL = 5,         /* NCCL error; outputs undefined */
    TRPLK_ENOMEM = 6         /* device allocation failed; outputs undefined */
} trplk_status;

typedef struct trplk_ctx trplk_ctx; /* opaque */

/* Device allocator hooks (the Python binding routes them to torch's caching allocator). */
typedef struct {
    void* (*alloc)(size_t bytes, void* user);
    void (*free)(void* ptr, void* user);
    void* user;
} trplk_allocator;

/* Row (z-slab) partition across ranks, SURVEY 8(e).  NULL => one GPU holding all rows.
 * nccl_unique_id points to the 128-byte ncclUniqueId that rank 0 generated (trplk_nccl_unique_id)
 * and the caller broadcast with its process group. */
typedef struct {
    int rank, nranks;
    int64_t row_begin, row_end;
    const void* nccl_unique_id;
} trplk_dist;

typedef struct {
    uint64_t seed;      /* start block rand(n,p^) seed, PAPER.md:509 (default 12); R13 */
    int max_cycles;     /* PAPER.md:509 (default 5000) */
    int tol_mode;       /* 0 ABS: ||A x - theta B x||_2 <= tol (Alg.1 step 12, default);
                           1 FROB: <= tol*||A||_F (eq 5.1); R8 */
    int restart_size;   /* p^ >= p kept at restart; 0 => p (R5) */
    int lock_mode;      /* 0 IF (one lock per cycle, Alg.1 step 12, R7); 1 WHILE */
    int debug_checks;   /* bit 1 (value 2): force the third CGS pass (R3) -- tests of that path */
    int use_graphs;     /* 1 (default): one CUDA graph per cycle; 0: eager launches */
    int precond;        /* 0 (default): Jacobi M on A - sigma B (R12); 1: none, M = I -- with
                           k_plus = 0 the thick-restart Lanczos baseline (eq 2.1, PAPER.md:77-80,
                           "cannot use preconditioning directly"), with m = 1, p = k_plus = 1 LOPCG;
                           2: Jacobi of A - rho_i B with the cycle's shift rho_i ("M may change at
                           every cycle with the goal to approximate (A - rho_i I)^-1", PAPER.md:171;
                           NEXT-2, reading P2c); not with block > 1 */
    int block;          /* b = 1 (default): Algorithm 1.  2..8: block TRPL+K ("A block
                           TRPL+K is also possible"; reading B1 of DESIGN.md): the inner space is the
                           block Krylov space of eq 3.2's C from the seeds M r_t .. M r_{t+b_e-1}
                           (b_e = min(b, p^-t+1, m)), built b vectors per SpMM; B = I, one rank */
} trplk_options;

typedef struct {
    int64_t a_matvecs;       /* A applications incl. verification ("MV", R18) */
    int64_t b_matvecs;       /* B applications (0 when B = I) */
    int64_t precond_applies; /* Jacobi applications */
    int64_t cycles;          /* outer cycles (restarts) */
    int64_t inner_steps;     /* inner Lanczos steps (eq 3.1) */
    int64_t verify_matvecs;  /* final verification A applications (R9), included in a_matvecs */
    int64_t random_draws;    /* stream-2 replacement vectors (R16) */
    int status;              /* trplk_status of the solve */
    double solve_seconds;    /* device time of the solve (CUDA events) */
    double model_bytes;      /* algorithmic HBM bytes of the solve (DESIGN.md byte model) */
    int64_t kernel_launches; /* device kernels launched by the solve (graph nodes included) */
} trplk_stats;

/* Fill *opt with the defaults documented above. */
void trplk_options_default(trplk_options* opt);

/* Write a fresh ncclUniqueId (128 bytes) into out (rank 0 calls this, then broadcasts). */
trplk_status trplk_nccl_unique_id(void* out, size_t out_bytes);

/* Create a context for the pencil (A, B) with the Jacobi preconditioner
 *   M = diag(max(|A_ii - sigma B_ii|, 1e-8 max_j |A_jj|))^-1      (reading R12)
 * n_global: order of A.  a_*: this rank's rows of A in CSR (host memory).
 * b_*: same for B, or all three NULL for B = I.  Every row must store its diagonal
 * entry (it may be zero).  Errors: EINVAL for a row range that does not tile n,
 * column ids out of range / not strictly increasing, q limits; ECUDA/ENCCL/ENOMEM.
 * Device formats: DIA (values per diagonal offset) when the local rows hold <= 32 distinct
 * offsets with <= 25 % padding and a contiguous ghost tail (stencils), else SELL-32 (diagonal
 * first).  Create is one parallel scan of the CSR; pinned host arrays are copied and scattered
 * into DIA on the device, pageable ones on the host. */
trplk_status trplk_create(trplk_ctx** out, int64_t n_global,
                          const int64_t* a_rowptr, const int64_t* a_col, const double* a_val,
                          const int64_t* b_rowptr, const int64_t* b_col, const double* b_val,
                          double sigma, const trplk_dist* dist, const trplk_allocator* alloc,
                          void* stream);

/* Run Algorithm 1 for the p smallest eigenpairs with max basis q = max_basis and l = k_plus
 * previous Ritz vectors (m = q - p^ - l >= 1 inner steps per cycle, reading R5).
 *   eigenvalues    [p]            host, ascending theta_1..theta_p
 *   eigenvectors   [n_local x p]  column-major, ld = n_local; device OR host pointer
 *                                 (cudaMemcpyDefault); B-orthonormal
 *   residual_norms [p]            host, ||A x_i - theta_i B x_i||_2 with ||x_i||_B = 1
 *   opt            NULL => defaults;  stats nullable.
 * Returns OK, NOT_CONVERGED or BREAKDOWN (outputs filled), else an error code. */
trplk_status trplk_solve(trplk_ctx* ctx, int p, int max_basis, int k_plus, double tol,
                         double* eigenvalues, double* eigenvectors, double* residual_norms,
                         const trplk_options* opt, trplk_stats* stats);

/* PL+1, Algorithm 2 (alg:pl+1) for the LOWEST eigenpair
 * of the context's pencil with the context's Jacobi preconditioner M ~ (A - sigma B)^-1 (or
 * M = I when use_precond = 0), readings P1-P6 of DESIGN.md section 2:
 *   step 4  G_k: B-orthonormal (CGS2) basis of span{M(A-rho_k B)x_k, ..., [M(A-rho_k B)]^m x_k}
 *   step 5  lowest primitive Ritz pair of (Q^T A Q, Q^T B Q), Q = [x_k, G_k, p_{k-1}], by
 *           Cholesky reduction + the Jacobi eig (p_{k-1} dropped when numerically dependent)
 *   step 6  x_{k+1} = Q w / ||Q w||_B, rho_{k+1} = x^T A x / x^T B x, r_{k+1} = (A - rho B) x
 *   step 7  p_k = B-normalised g_k - [p^T(A - rho_{k-1}B)g_k / p^T(A - rho_{k-1}B)p] p_{k-1}
 *           (variant 0, the paper's), or g_k + w(m+2) p_{k-1} (variant 1)
 * until ||r_k||_2 <= tol or max_iter iterations.  1 <= m <= 32.  Several ranks: the context's
 * row slabs, halo exchanges and rank-ordered reductions as trplk_solve (same result on every
 * rank; x_out holds this rank's rows).
 *   x0          start vector [n_local] (device or host), NULL: x0(i) = u01(seed, 3, i) (R13)
 *   rho         host: final rho_k;  resid: host ||r_k||_2;  x_out [n_local] device or host
 *               (cudaMemcpyDefault) or NULL: the B-normalised x_k
 *   log_*       host arrays of capacity log_cap (any NULL): rho_k, ||r_k||, and the step-7
 *               defect p_{k-1}^T(A - rho_{k-1}B)p_k / ||A||_F of the update that produced p_k
 *               (entry k+1), per iteration; *log_len = entries written
 * stats: a_matvecs, b_matvecs, cycles (= iterations), status, solve_seconds are filled.
 * Returns OK, NOT_CONVERGED, BREAKDOWN (Cholesky of Q^T B Q failed on x_k or G_k), EINVAL. */
trplk_status trplk_pl1_solve(trplk_ctx* ctx, int m, double tol, int variant, int use_precond, int max_iter,
                             uint64_t seed, const double* x0, double* rho, double* resid, double* x_out,
                             int log_cap, double* log_rho, double* log_res, double* log_conj, int* log_len,
                             trplk_stats* stats);

/* PL+1 global quasi-optimality diagnostic (Definition defnglbopt; reading P7
 * of DESIGN.md).  trplk_pl1_set_qopt(ctx, cap), 0 <= cap <= 64 (0 = off, the default), arms it
 * for the context's later trplk_pl1_solve calls: entry k < cap records rho(y*_k), the minimum of
 * the Rayleigh quotient over U_k = span{x_0} + span{g_0, ..., g_{k-1}} (g_k of
 * Alg. 2 step 6), from a B-orthonormal basis of U_k kept on the device (CGS2_B; g_k dropped on
 * the R16 breakdown test) and the lowest eigenvalue of Z^T A Z (the Jacobi eig kernel).  Costs,
 * per iteration, one CGS2_B, one A-SpMV and one Gram column (eager launches between the
 * iteration graphs, not counted in stats), plus 8 n_local x cap bytes of device memory.
 * Returns EINVAL for cap outside [0, 64].
 * trplk_pl1_get_qopt: of the last PL+1 solve, entries k = 0 .. ret-1 (ret <= cap):
 *   rho_star[k] = rho(y*_k);  dim[k] = dim U_k;  ratio[k] = (rho_k - rho(y*_k)) / (rho_k - lambda1),
 *   NaN where rho_k <= lambda1 (lambda1 = NaN: the solve's last rho_k).  Any pointer may be NULL
 *   (host arrays).  Returns 0 when the diagnostic was off. */
trplk_status trplk_pl1_set_qopt(trplk_ctx* ctx, int cap);
int trplk_pl1_get_qopt(const trplk_ctx* ctx, int cap, double lambda1, double* rho_star, int* dim, double* ratio);

/* Per-cycle log of the last solve (SURVEY 8(c.2) "Log per cycle"); any pointer may be NULL.
 * Arrays have capacity cap (thetas: cap x p^, row-major).  Returns the number of cycles logged. */
int trplk_get_log(const trplk_ctx* ctx, int cap, int* t, int64_t* mv, double* theta_t,
                  double* res, int* k, int* nprev, double* thetas);

/* Local problem facts: n_local, n_ghost, rank, nranks, ||A||_F, SELL bytes of A and B. */
trplk_status trplk_info(const trplk_ctx* ctx, int64_t* n_local, int64_t* n_ghost, int* rank,
                        int* nranks, double* frob_a, int64_t* sell_bytes_a, int64_t* sell_bytes_b);

void trplk_destroy(trplk_ctx* ctx);
const char* trplk_last_error(const trplk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TRPLK_H */
