/*
 * TRPL+K CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct fp64 implementation of Algorithm 1
 * (alg:trpl+k) with the readings R1-R20 of SURVEY.md 8(c.3)
 * and DESIGN.md.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  It shares no code with the
 * CUDA path (paper_1711_10128_b200/csrc) and neither includes the other.
 *
 * Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".
 */
#ifndef TRPLK_ORACLE_H
#define TRPLK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Counter-based U[0,1) generator, reading R13 (independent implementation). */
double orc_u01(uint64_t seed, uint64_t stream, uint64_t index);

/* y = A x, CSR in row order (eq 3.1 first line). */
void orc_spmv(int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
              const double* x, double* y);
/* x^T y with blocked fixed-order summation (4096-row blocks, pairwise across blocks). */
double orc_dot(int64_t n, const double* x, const double* y);
/* sqrt(sum of squares of all stored values) (eq 5.1 ||A||_F). */
double orc_frobenius(int64_t nnz, const double* val);
/* Jacobi preconditioner M_i = 1/max(|A_ii - sigma B_ii|, floor*max_j|A_jj|) (R12). */
void orc_jacobi_diag(int64_t n, const int64_t* a_rowptr, const int64_t* a_col, const double* a_val,
                     const int64_t* b_rowptr, const int64_t* b_col, const double* b_val,
                     double sigma, double floor_rel, double* M);
/* Small symmetric eig by cyclic-by-row Jacobi; T is k x k column-major (lda=k),
 * symmetrised first.  theta ascending, stable on ties, Y column-major k x k with the
 * largest-magnitude entry of each column positive (R10, R11). Returns sweeps used, <0 on failure. */
int orc_sym_eig(int k, const double* T, double* theta, double* Y);

/* CGS2 in the B-inner product (R3): w <- w - V V^T B w twice (+1 pass if the second pass
 * drops the norm by more than 1/sqrt2).  V is n x k column-major (ld = n).  B may be NULL.
 * Returns the final B-norm in *beta (w is NOT normalised), the coefficients of the passes
 * summed into h (k, may be NULL) and 1 on breakdown (final norm < 1e-14 * input norm). */
int orc_cgs2(int64_t n, int k, const double* V, double* w, const int64_t* b_rowptr,
             const int64_t* b_col, const double* b_val, double* h, double* beta, int* passes);

/* Xn(:,0:ncol) = U(:,0:k) Y(0:k,0:ncol), plain triple loop. Column-major, ld n / ldy. */
void orc_rotate(int64_t n, int k, const double* U, const double* Y, int ldy, int ncol, double* Xn);

typedef struct {
    int64_t n;
    const int64_t* a_rowptr; const int64_t* a_col; const double* a_val;
    const int64_t* b_rowptr; const int64_t* b_col; const double* b_val;  /* all NULL: B = I */
    double sigma;
    int p, q, l;            /* wanted pairs, max basis, k_plus */
    double tol;
    int tol_mode;           /* 0 ABS: ||r|| <= tol; 1 FROB: ||r|| <= tol*||A||_F (eq 5.1) */
    uint64_t seed;
    int max_cycles;
    int restart_size;       /* p^ (>= p); 0 -> p */
    int lock_mode;          /* 0 IF (Alg. 1 step 12, R7), 1 WHILE */
    int debug;              /* 1: log ||T - U^T A U||_max and ||U^T B U - I||_max per cycle */
    int precond;            /* 0 Jacobi (R12); 1 none, M = I: with l = 0 thick-restart Lanczos (eq 2.1,
                               PAPER.md:77-80), with m = p = l = 1 LOPCG (eq 2.2 with p = 1);
                               2 Jacobi of A - rho_i B re-formed every cycle (reading P2c);
                               3 IC(0) of A - sigma B ("incomplete ... factorization", P2a) */
    int block;              /* b <= 8: block TRPL+K ("A block TRPL+K is also possible", reading
                               B1): the inner space is the block Krylov space of eq 3.2's operator C
                               (one shift rho = theta_t) from the b_e = min(b, p^-t+1, m) seeds
                               M r_t .. M r_{t+b_e-1}; 0/1 = Algorithm 1 */
} orc_problem;

typedef struct {
    int status;             /* 0 OK, 2 NOT_CONVERGED, 3 BREAKDOWN, 1 EINVAL */
    int cycles;
    int64_t a_matvecs, b_matvecs, precond_applies, verify_matvecs, inner_steps, random_draws;
    /* per-cycle log; arrays of capacity log_cap (caller-owned, may be NULL) */
    int log_cap, log_len;
    int* log_t;             /* target (1-based) at the RR of the cycle */
    int64_t* log_mv;        /* cumulative A-matvecs at the end of the cycle */
    double* log_theta_t;    /* theta_t at the RR */
    double* log_res;        /* ||r_t|| at the RR */
    int* log_k;             /* basis width at the RR */
    int* log_nprev;         /* X^prev columns appended this cycle */
    double* log_thetas;     /* log_cap x p^ Ritz values theta_1..p^ */
    double* log_terr;       /* debug: max |T - U^T A U| */
    double* log_orth;       /* debug: max |U^T B U - I| */
    /* optional dumps for tiny problems: X at the start of cycle c (c < dump_cycles) */
    int dump_cycles;
    double* dump_X;         /* dump_cycles x (n x p^) */
    double* dump_rho;       /* dump_cycles */
    int* dump_t;            /* dump_cycles */
    /* optional samples of the returned eigenvectors (large problems): sample_vals[i + n_sample*c]
     * = x_c(sample_rows[i]) for c < p */
    int n_sample;
    const int64_t* sample_rows;
    double* sample_vals;
    int verbose;            /* 1: one progress line per cycle on stderr */
} orc_report;

/* Inner steps of eq 3.1 alone (the code orc_trplk_solve runs for step j < m): for j < nsteps,
 * g = U(:,k0+j-1): z = A g, T(0:k0+j, k0+j-1) = U^T z (mirrored, ldT), w = M(z - rho B g), CGS2_B of w
 * against U(:,0:k0+j), U(:,k0+j) = w/beta.  U is n x (k0+nsteps) column-major with orthonormal
 * U(:,0:k0); M the Jacobi diagonal; work: caller scratch of 4n doubles (NULL: allocated here).  Returns the steps run (fewer after a breakdown).  Used by
 * bench.py to time a bounded sample of the oracle at sizes where a full solve takes hours. */
int orc_inner_steps(const orc_problem* P, const double* M, double rho, double* U, int k0, int nsteps,
                    double* T, int ldT, double* work /* 4n scratch, or NULL */);

/* IC(0) factor L (CSR: rows ascending by column, the diagonal last) of A - sigma B on A's lower
 * pattern (reading P2a, see oracle.c).  Returns nnz(L); copies into the outputs when cap >= nnz. */
int64_t orc_ic0(const orc_problem* P, double sigma, int64_t* rp_out, int64_t* ci_out, double* val_out, int64_t cap);

/* Algorithm 1 in full.  evals[p], resid[p] ascending; evecs n x p column-major. */
int orc_trplk_solve(const orc_problem* prob, double* evals, double* evecs, double* resid,
                    orc_report* rep);

/* ------------------------------------------------------------------ PL+1 (Algorithm 2)
 * Preconditioned Lanczos+1 for the lowest eigenpair of (A, B) (alg:pl+1),
 * readings P1-P6 of DESIGN.md section 2 (NEXT-1 of SURVEY 8(f)). */
typedef struct {
    int64_t n;
    const int64_t* a_rowptr; const int64_t* a_col; const double* a_val;
    const int64_t* b_rowptr; const int64_t* b_col; const double* b_val;  /* all NULL: B = I */
    double sigma;           /* M = Jacobi of A - sigma B (R1, R12 floor) */
    int use_precond;        /* 0: M = I */
    int m;                  /* Krylov block size (step 4), 1..32 */
    double tol;             /* delta: stop when ||r_k||_2 <= delta (step 3) */
    uint64_t seed;          /* x_0(i) = u01(seed, 3, i) when x0 is NULL (P6) */
    const double* x0;       /* optional start vector (n) */
    int max_cycles;
    int variant;            /* 0: step-7 conjugation (paper); 1: practical p = g + p w(m+2) */
} orc_pl1_problem;

typedef struct {
    int status;             /* 0 OK, 2 NOT_CONVERGED, 3 BREAKDOWN, 1 EINVAL */
    int cycles;             /* outer iterations performed */
    int64_t a_matvecs, b_matvecs;
    double rho, resid;      /* final rho_k and ||r_k||_2 */
    int log_cap, log_len;   /* per-iteration log, entry k = state at the top of iteration k */
    double* log_rho;        /* rho_k = rho(x_k) */
    double* log_res;        /* ||r_k||_2 */
    double* log_conj;       /* p_{k-1}^T (A - rho_{k-1} B) p_k / ||A||_F of the step-7 update that
                               produced p_k (entry k+1 holds iteration k's); 0 where undefined */
    double* log_ritz;       /* lowest Ritz value of step 5 at iteration k (entry k), or 0 */
    int* log_mg;            /* columns of G_k built at iteration k (entry k; < m after a breakdown) */
    int* log_nq;            /* columns of Q_k used in the RR at iteration k (p dropped if dependent) */
    /* Global quasi-optimality diagnostic (Definition defnglbopt; reading P7):
     * U_k = span{x_0} + W_k, W_k = span{g_0, ..., g_{k-1}}.  Entry k (k <
     * qopt_cap): log_qopt[k] = rho(y*_k), the minimum of the Rayleigh quotient over U_k;
     * log_qdim[k] = dim U_k as built (g_j B-orthonormalised by CGS2 against the earlier basis and
     * dropped when dependent, the R16 threshold).  log_g (optional, n x qopt_cap column-major):
     * column k = g_k of step 6.  qopt_cap = 0: off.  The diagnostic's matvecs are not counted. */
    int qopt_cap;
    double* log_qopt;
    int* log_qdim;
    double* log_g;
} orc_pl1_report;

/* Algorithm 2.  x_out (n, may be NULL): the final B-normalised iterate. */
int orc_pl1_solve(const orc_pl1_problem* prob, double* x_out, orc_pl1_report* rep);

#ifdef __cplusplus
}
#endif
#endif
