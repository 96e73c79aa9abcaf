/*
 * trplk_kernels.h -- kernel-level entry points of libtrplk.so (parity tests,
 * diagnostics).  Each call runs exactly the device kernels trplk_solve uses for
 * that step, on caller-provided device buffers, on the context's stream, and
 * synchronises before returning host outputs.  Vectors that are multiplied by A
 * or B (the `x`/`g` arguments) must hold n_local + n_ghost entries: the ghost
 * tail (global columns owned by other ranks, ascending global id) is filled by
 * the caller.  U blocks are column-major with leading dimension ldu >= n_local.
 * Errors: EINVAL on bad sizes (k > TRPLK_MAX_BASIS, ld too small), ECUDA.
 */
#ifndef TRPLK_KERNELS_H
#define TRPLK_KERNELS_H

#include "trplk.h"

#ifdef __cplusplus
extern "C" {
#endif

/* y = Op x on the local rows, Op = A (which=0) or B (which=1).  S1, eq 3.1 line 1. */
trplk_status trplk_k_spmv(trplk_ctx* ctx, int which, const double* x, double* y);

/* Fused inner-step kernel K1 (eq 3.1 + preconditioner, reading R1):
 *   z = A g,  s = B g,  w = M (z - rho s)   -> w (device, n_local)
 *   tcol[0:k] = U^T z                         (T(1:k, k) of eq 3.1)
 *   h1[0:k]   = U^T (B w),  wnorm2 = w^T B w  (first CGS2 pass coefficients, R3)
 * For B != I the B-products come from the second kernel the solver runs (B-SpMV + dots). */
trplk_status trplk_k_step1(trplk_ctx* ctx, const double* U, int64_t ldu, int k, const double* g,
                           double rho, double* w, double* tcol, double* h1, double* wnorm2);

/* CGS2 in the B-inner product of w against U(:,0:k) (reading R3), device path:
 * out = (w - U h)/beta with h the summed pass coefficients (host, k entries), beta the
 * final B-norm, breakdown = final norm < 1e-14 ||w||_B, passes = 2 or 3.
 * On breakdown out is left unnormalised. */
trplk_status trplk_k_cgs2(trplk_ctx* ctx, const double* U, int64_t ldu, int k, const double* w,
                          double* out, double* h, double* beta, int* breakdown, int* passes);

/* Block kernel of the +K augmentation (block.cuh; Alg.1 steps 6-8), c <= 8
 * vectors against U(:,0:k) in one pass over U:
 *   mode 0 GRAM  HV = U^T Y (k x c),            G = Y^T Y (c x c)
 *   mode 1 UPD   Q = Y Rinv (Rinv: c x c upper triangle, NULL = I), Y' = Q - U H -> Yout (device,
 *                may alias Y), HV = U^T Y', G = Y'^T Y'      (H: k x c host, required)
 *   mode 2 SPMM  HV = U^T (A Y)   (Y with ghost tails; G not written)
 * Host matrices column-major with leading dimension = their row count (HV: k, G/Rinv: c, H: k).
 * Errors: EINVAL (c outside 1..8, k > 64, lds, missing H/Yout for UPD), ECUDA. */
trplk_status trplk_k_block(trplk_ctx* ctx, int mode, const double* U, int64_t ldu, int k, const double* Y,
                           int64_t ldy, int c, const double* Rinv, const double* H, double* Yout, int64_t ldyo,
                           double* HV, double* G);

/* X(:,0:ncol) = U(:,0:k) Y(0:k,0:ncol) with the fp64 DMMA kernel (Alg.1 steps 11/15,
 * PAPER.md:193,198).  Y host, column-major k x ncol (ncol <= 24). */
trplk_status trplk_k_rotate(trplk_ctx* ctx, const double* U, int64_t ldu, int k, const double* Y,
                            int ncol, double* X, int64_t ldx);

/* One-CTA parallel-ordered cyclic Jacobi of sym(T), k x k column-major host arrays
 * (Alg.1 step 11; R10/R11 ordering and sign rule). */
trplk_status trplk_k_sym_eig(trplk_ctx* ctx, int k, const double* T, double* theta, double* Y);

/* Timing of the Rayleigh-Ritz kernel alone (measurement): the one-CTA Jacobi of sym(T) (k x k,
 * column-major host array) launched `reps` times back to back on the context's stream, timed
 * with CUDA events.  *ms = average device milliseconds per launch, *sweeps = Jacobi sweeps the
 * last launch took (nullable).  Errors: EINVAL (k, reps), ECUDA. */
trplk_status trplk_k_sym_eig_time(trplk_ctx* ctx, int k, const double* T, int reps, double* ms, int* sweeps);

/* r = A x - theta B x (Alg.1 step 12), u = M r (step 15 seed), rnorm2 = ||r||^2. */
trplk_status trplk_k_residual(trplk_ctx* ctx, const double* x, double theta, double* r, double* u,
                              double* rnorm2);

/* x[i] = U01(seed, stream, col*n_global + global_row(i)) for the local rows (reading R13). */
trplk_status trplk_k_random(trplk_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t col, double* x);

/* Host-only halo planning of a row slab (no device work; the code trplk_create runs).
 *   ghosts_out[cap]  sorted unique global column ids outside [row_begin,row_end) referenced by the
 *                    local rows of A (and B, may be NULL); the ghost tail of every local vector
 *   owners_out[cap]  owner rank of each ghost given ranges[2*nranks] = {begin_r, end_r} (rank order)
 *   *n_ghost         count (set even when cap is too small, which returns EINVAL)
 * Local column id of a global column c: c - row_begin if owned, else n_local + index in ghosts_out. */
trplk_status trplk_plan_ghosts(int64_t row_begin, int64_t row_end, const int64_t* a_rowptr, const int64_t* a_col,
                               const int64_t* b_rowptr, const int64_t* b_col, const int64_t* ranges, int nranks,
                               int64_t* ghosts_out, int* owners_out, int64_t cap, int64_t* n_ghost);

/* Debug switches of the context (tests of rare paths).  Bit 0: take the third CGS pass
 * (reading R3) in every CGS2 even when the second pass kept more than 1/sqrt2 of the norm -- the
 * same arithmetic as a genuine third pass, so its kernels can be checked against the oracle.
 * trplk_options.debug_checks bit 1 does the same for one solve.  Bit 1: run the m inner steps
 * of every cycle as ONE cooperative grid-wide kernel (inner_grid.cuh; one CTA per SM, grid
 * barriers and all-reduces instead of kernel boundaries) where it applies -- one rank, B = I,
 * max_basis <= 32, n above the single-CTA small path; also enabled by the environment variable
 * TRPLK_GRID=1.  Same readings (R1, R3, R16) as the multi-kernel step.  Errors: EINVAL (ctx NULL). */
trplk_status trplk_set_debug(trplk_ctx* ctx, int flags);

/* Host-staged rank exchanges (test infrastructure and single-GPU multi-process runs): collective
 * callbacks every rank calls in the same order on HOST buffers; each returns 0 on success.
 *   allgather  recv[r*bytes .. (r+1)*bytes) <- rank r's send, for every rank r
 *   sendrecv   grouped point-to-point: send_buf[i] (send_bytes[i]) to send_peer[i], recv_buf[j]
 *              (recv_bytes[j]) from recv_peer[j]; every send matches the peer's recv of the same size
 *   allreduce  v[0:count] <- elementwise sum (op 0) or max (op 1) over ranks (create time only) */
typedef struct {
    int (*allgather)(const void* send, void* recv, size_t bytes, void* user);
    int (*sendrecv)(int nsend, const int* send_peer, const void* const* send_buf, const size_t* send_bytes,
                    int nrecv, const int* recv_peer, void* const* recv_buf, const size_t* recv_bytes, void* user);
    int (*allreduce)(double* v, int count, int op, void* user);
    void* user;
} trplk_host_comm;

/* trplk_create whose row-partition exchanges go through an in-process loopback hub
 * (loopback_hub, from trplk_loopback_create) or host callbacks (host_comm) instead of NCCL; exactly
 * one of the two must be non-NULL, dist must be given (dist->nccl_unique_id is ignored).  Solves on
 * such contexts run eagerly (no CUDA graphs: the exchanges are host rendezvous).  Otherwise the
 * arguments, ownership and errors of trplk_create. */
trplk_status trplk_create_ex(trplk_ctx** out, int64_t n_global, const int64_t* a_rowptr, const int64_t* a_col,
                             const double* a_val, const int64_t* b_rowptr, const int64_t* b_col, const double* b_val,
                             double sigma, const trplk_dist* dist, void* loopback_hub,
                             const trplk_host_comm* host_comm, const trplk_allocator* alloc, void* stream);

/* In-process loopback hub for nranks ranks (test infrastructure): pass it to
 * every rank's trplk_create_ex, one host thread per rank, all on the same
 * GPU.  Every exchange (halo planes, reduction partials, create-time plans) becomes a rendezvous
 * of the rank threads with device-to-device copies on the receiving rank's stream ordered by
 * CUDA events -- no kernel waits on another rank.  Solves on loopback ranks run eagerly (no
 * CUDA graphs).  Destroy the hub after every rank's context.  Errors: EINVAL (nranks < 1). */
trplk_status trplk_loopback_create(int nranks, void** hub);
void trplk_loopback_destroy(void* hub);

/* Live profile of the inner step (measurement): while enabled, every
 * outer cycle records CUDA events around the three kernel groups of its middle inner step
 *   [0] K1  fused SpMV + preconditioner + T-column/h1 dots
 *   [1] K2  CGS pass 2 (update + dots; for B != I the B-SpMV dot passes and the update)
 *   [2] K3  final update + normalisation (+ gated third-pass fix-up)
 * and accumulates their device milliseconds and algorithmic bytes (byte model of DESIGN.md).
 * enable=1 clears the accumulators.  read: ms[3], bytes[3] sums over `count` cycles. */
trplk_status trplk_profile(trplk_ctx* ctx, int enable);
trplk_status trplk_profile_read(const trplk_ctx* ctx, double* ms, double* bytes, int64_t* count);
/* Cycle-phase breakdown of the live profile: device ms summed over `count` profiled cycles of
 *   [0] seed CGS2 (R4)  [1] the m inner steps (eq 3.1)  [2] +K (Alg.1 steps 6-8)
 *   [3] Rayleigh-Ritz eig (step 11)  [4] rotation U Y (steps 11/15)  [5] residual of the target
 * (events at the phase boundaries inside every cycle).  Errors: EINVAL (ctx NULL). */
trplk_status trplk_profile_phases(const trplk_ctx* ctx, double* ms, int64_t* count);
/* Demangled names of the kernels that ran the three profiled groups (K1;K2;K3, ';'-separated;
 * an empty field where the group is fused into K1), written NUL-terminated into buf[len].
 * Errors: EINVAL (NULL ctx/buf or len too small). */
trplk_status trplk_profile_kernels(const trplk_ctx* ctx, char* buf, size_t len);

#ifdef __cplusplus
}
#endif
#endif
